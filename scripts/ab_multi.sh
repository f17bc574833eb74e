# A/B/C... of library builds and environment settings on one box:
#   ab_multi.sh "LIB|ENV" "LIB|ENV" ...   (ENV may be empty), three rounds
for i in 1 2 3; do for spec in "$@"; do
  lib=${spec%%|*}; envs=${spec#*|}
  HGPU_LIB=$lib env $envs python bench.py --steps 5 --warmup 3 --no-lambda --no-cpu-baseline --no-secondary > gpurun_out/sw.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('$spec', round(d['ms_per_step'],1), d['parity']['bit_exact'])" || tail -3 gpurun_out/sw.json
done; done
