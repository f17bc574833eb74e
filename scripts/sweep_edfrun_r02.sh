# EDF run length (panels per k_update_tiled launch) and the chain-only floor
# (deferred update skipped, timing-experiments build) on one box
run() { env $1 python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('[$1]', round(d['ms_per_step'],1), d['parity']['bit_exact'], round(d['roofline']['frac'],3), round(d['roofline']['update_share_of_step'],3))" || tail -3 gpurun_out/sw.err; }
for i in 1 2; do
for v in "A=1" "HGPU_EDF_RUN=4" "HGPU_EDF_RUN=3" "HGPU_EDF_RUN=2" "HGPU_EDF_RUN=2 HGPU_SM_SPLIT=2:b" "HGPU_EDF_RUN=4 HGPU_SM_SPLIT=2:b" "HGPU_SM_SPLIT=2:b"; do run "$v"; done
done
run "HGPU_LIB=paper_0902_0852_b200/libhgpu_exp.so HGPU_DEBUG=512"
run "HGPU_LIB=paper_0902_0852_b200/libhgpu_exp.so HGPU_DEBUG=512 HGPU_SM_SPLIT=2:b"
