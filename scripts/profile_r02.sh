# Round-2 evidence (one B200): the default bench line, the ncu launch list of
# a short bench, and full captures of one in-step k_update_tiled (EDF run)
# and one k_pivot.
set -e
out=gpurun_out
python bench.py > $out/bench_final.log 2>&1
python bench.py --steps 2 --warmup 1 --no-lambda --no-cpu-baseline --no-secondary > $out/bench_short.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_r02.csv \
  python bench.py --steps 2 --warmup 1 --no-lambda --no-cpu-baseline --no-secondary > $out/ncu_launches.log 2>&1
python scripts/factor_x1.py 1 > $out/fx1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_tiled --launch-skip 60 --launch-count 1 \
  -o $out/k_update_r02 -f python scripts/factor_x1.py 1 > $out/ncu_update.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_pivot$" --launch-skip 500 --launch-count 1 \
  -o $out/k_pivot_r02 -f python scripts/factor_x1.py 1 > $out/ncu_pivot2.log 2>&1
echo done > $out/profile_done.txt
