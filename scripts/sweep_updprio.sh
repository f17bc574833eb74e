run() { env $1 python bench.py --steps 3 --warmup 3 --no-lambda --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('[$1]', round(d['ms_per_step'],1), d['parity']['bit_exact'], [(s['config'], round(s['ms_per_factorisation'],1), round(s['update_share'],3)) for s in d['secondary_configs']])" || tail -3 gpurun_out/sw.err; }
for v in "HGPU_UPD_PRIO=0" "HGPU_UPD_PRIO=2" "HGPU_UPD_PRIO=5" "HGPU_UPD_PRIO=5 HGPU_FAR_PRIO=2"; do run "$v"; done
