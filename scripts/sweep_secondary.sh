# configs 4 and 5 (bench.py's secondary_configs) under schedule variants
run() { env $1 python bench.py --steps 2 --warmup 3 --no-lambda --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('[$1]', round(d['ms_per_step'],1), [(s['config'], round(s['ms_per_factorisation'],1), round(s['update_share'],3)) for s in d['secondary_configs']])" || tail -3 gpurun_out/sw.err; }
for v in "A=1" "HGPU_FAR_LANES=2 HGPU_GRID=2" "HGPU_FAR_LANES=4" "HGPU_GRID=2" "HGPU_FAR_LANES=2" "HGPU_NEAR=40" "HGPU_FAR_SUB=16"; do run "$v"; done
