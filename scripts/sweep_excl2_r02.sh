# chain + near rows on an exclusive group of SMs (panel stream on group a)
for v in "HGPU_SM_SPLIT=32:a" "HGPU_SM_SPLIT=48:a" "HGPU_SM_SPLIT=64:a" "HGPU_SM_SPLIT=32:a HGPU_NEAR=48" "HGPU_SM_SPLIT=48:a HGPU_NEAR=96"; do
  env $v python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), d['parity']['bit_exact'])" || tail -3 gpurun_out/sw.json
done
rm -f gpurun_out/tl_4b.txt; HGPU_SM_SPLIT=4:b HGPU_TIMELINE=gpurun_out/tl_4b.txt python scripts/factor_x1.py 2 > /dev/null 2>&1
