# green-context SM partitions after the reciprocal change (one B200)
for v in "" "HGPU_SM_SPLIT=8" "HGPU_SM_SPLIT=16" "HGPU_SM_SPLIT=8:b" "HGPU_SM_SPLIT=16:b" "HGPU_SM_SPLIT=8:p" "HGPU_SM_SPLIT=24:a"; do
  env $v python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), d['parity']['bit_exact'])" || tail -3 gpurun_out/sw.json
done
