for v in "" "HGPU_FAR_LANES=3" "HGPU_FAR_LANES=4" "HGPU_FAR_SUB=4" "HGPU_FAR_SUB=16" "HGPU_COL_EXTRACT=2" "HGPU_NEXT_ROW=1" "HGPU_SM_SPLIT=4:b" "HGPU_EDF=2"; do
  env $v python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), d['parity']['bit_exact'])" || tail -3 gpurun_out/sw.json
done
