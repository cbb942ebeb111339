#!/bin/bash
# A/B of body variants on the GPU box: fwd/bwd row loads in flight
# (HPS_FB_ROUNDS rebuild) x big-segment path on a side stream (HPS_BIG_SIDE).
cd "$(dirname "$0")/.."
run() { python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,2))"; }
for r in ${ROUNDS:-default 2}; do
  if [ "$r" = default ]; then make -s -B -C paper_2003_05622_b200/csrc >/dev/null 2>&1
  else make -s -B -C paper_2003_05622_b200/csrc EXTRA=-DHPS_FB_ROUNDS=$r >/dev/null 2>&1; fi
  for side in ${SIDES:-1 0}; do HPS_BIG_SIDE=$side run "rounds=$r side=$side"; HPS_BIG_SIDE=$side run "rounds=$r side=$side"; done
done
make -s -B -C paper_2003_05622_b200/csrc >/dev/null 2>&1
