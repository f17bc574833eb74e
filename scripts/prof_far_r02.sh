# full ncu captures of one far-row extraction and one far-row division (early stage, ~300 rows per lane)
out=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"^k_extract$" --launch-skip 4 --launch-count 1 \
  -o $out/k_extract_far -f python scripts/factor_x1.py 1 > $out/ncu_ex.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_divide$" --launch-skip 4 --launch-count 1 \
  -o $out/k_divide_far -f python scripts/factor_x1.py 1 > $out/ncu_dv.log 2>&1
