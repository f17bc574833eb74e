# ncu --set full of one k_pivot launch (stage 500 of config 3) and the
# timeline analyses of the pivot chain; summaries for profiles/.
set -u
out=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name k_pivot \
  --launch-skip 500 --launch-count 1 -o $out/prof_k_pivot -f \
  python scripts/factor_x1.py 1 > $out/prof_k_pivot.log 2>&1
ncu -i $out/prof_k_pivot.ncu-rep --page details --csv > $out/prof_k_pivot_details.csv 2>/dev/null
ncu -i $out/prof_k_pivot.ncu-rep --page raw --csv > $out/prof_k_pivot_raw.csv 2>/dev/null
rm -f $out/tl_final.txt
HGPU_TIMELINE=$out/tl_final.txt timeout 300 python scripts/factor_x1.py 1 > /dev/null 2>&1
python scripts/timeline.py $out/tl_final.txt > $out/tl_final_summary.txt 2>&1
python scripts/boundary2.py $out/tl_final.txt > $out/tl_final_boundary.txt 2>&1
python scripts/chain_deps.py $out/tl_final.txt > $out/tl_final_deps.txt 2>&1
HGPU_DEBUG=4096 timeout 300 python scripts/factor_x1.py 1 > $out/k_pivot_phases.txt 2>&1
