# bench variants after the reciprocal change (one B200): ms per step
for v in "" "HGPU_NEXT_ROW=1" "HGPU_NEAR=48" "HGPU_NEAR=96" "HGPU_FAR_LANES=3" "HGPU_PIVOT_THREADS=384" "HGPU_NEXT_ROW=1 HGPU_NEAR=96" "HGPU_EDF=2"; do
  env $v python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), d['parity']['bit_exact'])"
done
