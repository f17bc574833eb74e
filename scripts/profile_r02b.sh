# Round-2 final evidence (one B200): ncu launch list of ONE full config-3
# factorisation at x1 (every launch, serialised), and full captures of one
# k_pivot (stage 500) and one in-step k_update_tiled band run.
set -e
out=gpurun_out
python scripts/factor_x1.py 2 > $out/fx1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 13000 --csv --log-file $out/launches_factor_r02.csv \
  python scripts/factor_x1.py 1 > $out/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_pivot$" --launch-skip 500 --launch-count 1 \
  -o $out/k_pivot_r02b -f python scripts/factor_x1.py 1 > $out/ncu_pivot.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_tiled --launch-skip 150 --launch-count 1 \
  -o $out/k_update_r02b -f python scripts/factor_x1.py 1 > $out/ncu_update.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_rq_products --launch-count 1 \
  -o $out/k_rq_r02b -f python scripts/lambda_c3_ii.py > $out/ncu_rq.log 2>&1 || true
echo done > $out/profile_done.txt
