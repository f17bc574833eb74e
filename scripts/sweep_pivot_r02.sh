# k_pivot footprint (one B200): the 512-thread kernel needs a whole SM's
# registers; the 256-thread lean kernel fits beside two update CTAs
for v in "" "HGPU_PIVOT_THREADS=256" "HGPU_PIVOT_THREADS=256 HGPU_SM_SPLIT=8:b" "HGPU_PIVOT_THREADS=256 HGPU_NEXT_ROW=1"; do
  env $v python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],1), d['parity']['bit_exact'])" || tail -3 gpurun_out/sw.json
done
rm -f gpurun_out/tl256.txt
HGPU_PIVOT_THREADS=256 HGPU_TIMELINE=gpurun_out/tl256.txt python scripts/factor_x1.py 2 > /dev/null 2>&1
