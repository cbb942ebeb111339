#!/bin/bash
# A/B of runtime knobs on the GPU box: each argument is a space-free list of
# VAR=value pairs separated by commas ("-" = defaults); every variant runs
# REPS times (default 2), interleaved. Prints value, ms/step, e2e.
cd "$(dirname "$0")/.."
REPS=${REPS:-2}
for rep in $(seq 1 $REPS); do
  for v in "$@"; do
    envs=""; [ "$v" != "-" ] && envs=$(echo "$v" | tr ',' ' ')
    env $envs python bench.py --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,2))"
  done
done
