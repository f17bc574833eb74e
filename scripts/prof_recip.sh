# ncu --set full of one k_recip launch (config 3, x1, stage 50), with source.
out=gpurun_out
HGPU_SM_SPLIT=0 timeout 600 ncu --set full --clock-control none --import-source on \
  --kernel-name k_recip --launch-skip 50 --launch-count 1 -o $out/prof_k_recip -f \
  python scripts/factor_x1.py 1 > $out/prof_k_recip.log 2>&1
ncu -i $out/prof_k_recip.ncu-rep --page details --csv > $out/prof_k_recip_details.csv 2>/dev/null
ncu -i $out/prof_k_recip.ncu-rep --page source --csv --print-source cuda,sass > $out/prof_k_recip_sass.csv 2>/dev/null
