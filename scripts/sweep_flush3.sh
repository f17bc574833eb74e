run() { env $1 python bench.py --steps 2 --warmup 3 --no-lambda --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('[$1]', round(d['ms_per_step'],1), [(s['config'], round(s['ms_per_factorisation'],1), round(s['update_share'],3)) for s in d['secondary_configs']])" || tail -3 gpurun_out/sw.err; }
for v in "HGPU_SLOT_FRAC=0.6" "HGPU_SLOT_FRAC=0.75" "HGPU_SLOT_FRAC=0.85"; do run "$v"; done
