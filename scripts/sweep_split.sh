# Factorisation time (and optionally the timeline) under scheduling knobs.
# Usage: CASES="HGPU_SM_SPLIT=0 HGPU_NEAR=64|HGPU_SM_SPLIT=16:b" TL=1 bash scripts/sweep_split.sh
IFS='|' read -ra cases <<< "${CASES:-HGPU_SM_SPLIT=0}"
for c in "${cases[@]}"; do
  echo "== $c"
  env $c timeout 120 python scripts/factor_x1.py 2 2>&1 | tail -1
  if [ "${TL:-0}" = 1 ]; then
    f=gpurun_out/tl_$(echo $c | tr " =:" "_..").txt; rm -f $f
    env $c HGPU_TIMELINE=$f timeout 120 python scripts/factor_x1.py 1 > /dev/null 2>&1
    python scripts/timeline.py $f
  fi
done
