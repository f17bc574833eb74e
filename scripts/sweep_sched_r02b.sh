# schedule knobs re-swept after the register-ladder reciprocal (one box)
run() { env $1 python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('[$1]', round(d['ms_per_step'],1), d['parity']['bit_exact'], round(d['roofline']['frac'],3), round(d['roofline']['update_share_of_step'],3))" || tail -3 gpurun_out/sw.err; }
for i in 1 2; do
for v in "A=1" "HGPU_NEXT_ROW=1" "HGPU_COL_EXTRACT=1" "HGPU_NEAR=32" "HGPU_NEAR=40" "HGPU_FAR_LANES=3" "HGPU_FAR_SUB=16" "HGPU_PIVOT_SEGS=4" "HGPU_GRID=3"; do run "$v"; done
done
