run() { env $1 python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('[$1]', round(d['ms_per_step'],1), d['parity']['bit_exact'], round(d['roofline']['frac'],3), round(d['roofline']['update_share_of_step'],3))" || tail -3 gpurun_out/sw.err; }
python -c "import torch; print(torch.cuda.get_device_name(0))"
for i in 1 2; do
for v in "HGPU_FAR_PRIO=0 HGPU_PRE_NEAR=0" "HGPU_FAR_PRIO=1 HGPU_PRE_NEAR=0" "HGPU_FAR_PRIO=2 HGPU_PRE_NEAR=0" "HGPU_FAR_PRIO=0 HGPU_PRE_NEAR=1" "HGPU_FAR_PRIO=1 HGPU_PRE_NEAR=1" "HGPU_FAR_PRIO=2 HGPU_PRE_NEAR=1" "HGPU_FAR_PRIO=1 HGPU_PRE_NEAR=1 HGPU_FAR_LANES=2" "HGPU_FAR_PRIO=1 HGPU_PRE_NEAR=1 HGPU_FAR_LANES=4"; do run "$v"; done
done
