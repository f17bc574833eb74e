#!/bin/bash
# One GPU session: tests, bench, launch list, full profile of k_update_tiled.
set -u
out=gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -x -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/gpu_tests.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $out/bench_ref.json 2> $out/bench_ref.err
if [ "${NCU:-1}" = 1 ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-lambda > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name k_update_tiled \
  --launch-skip 20 --launch-count 1 -o $out/k_update_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-lambda > $out/ncu_full.log 2>&1
fi
tail -n 3 $out/gpu_tests.log; cat $out/bench.json; tail -n 2 $out/bench.err; cat $out/bench_ref.json; tail -n 2 $out/ncu_launch.log; tail -n 2 $out/ncu_full.log
