# Final-build evidence (one B200): launch list of ONE whole config-3
# factorisation at x1, and full captures of one k_pivot (stage 500) and of
# eight consecutive k_update_tiled launches (the longest is a full band run).
set -e
out=gpurun_out
python scripts/factor_x1.py 2 > $out/fx1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 16000 --csv --log-file $out/launches_factor_final.csv \
  python scripts/factor_x1.py 1 > $out/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_pivot$" --launch-skip 500 --launch-count 1 \
  -o $out/k_pivot_final -f python scripts/factor_x1.py 1 > $out/ncu_pivot.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_tiled --launch-skip 120 --launch-count 8 \
  -o $out/k_update_final -f python scripts/factor_x1.py 1 > $out/ncu_update.log 2>&1
echo done > $out/profile_done.txt
