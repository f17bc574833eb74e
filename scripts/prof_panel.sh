# ncu --set full of one far-row k_extract and one far-row k_divide launch
# (every third launch of each kernel is the far-row one; config 3, x1).
set -u
out=gpurun_out
for k in k_extract k_divide k_update_col; do
  HGPU_SM_SPLIT=0 HGPU_RATIO_GEMM=0 timeout 600 ncu --set full --clock-control none --import-source on \
    --kernel-name $k --launch-skip 32 --launch-count 1 -o $out/prof_$k -f \
    python scripts/factor_x1.py 1 > $out/prof_$k.log 2>&1
  ncu -i $out/prof_$k.ncu-rep --page details --csv > $out/prof_${k}_details.csv 2>/dev/null
  ncu -i $out/prof_$k.ncu-rep --page source --csv --print-source cuda > $out/prof_${k}_src.csv 2>/dev/null
done
