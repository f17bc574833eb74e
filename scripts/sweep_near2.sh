for i in 1 2; do for v in "HGPU_NEAR=32" "HGPU_NEAR=34" "HGPU_NEAR=36" "HGPU_NEAR=40" "HGPU_NEAR=48"; do
  env $v python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), d['parity']['bit_exact'])" || tail -3 gpurun_out/sw.json
done; done
