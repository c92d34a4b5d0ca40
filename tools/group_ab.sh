#!/bin/bash
# A/B of the trajectory-kernel configuration on config 2 (GPU box).
# usage: tools/group_ab.sh "4 8 16 32"
for g in ${1:-4 8 16 32}; do
  for st in on off; do
    if [ $st = off ]; then export SABER_NO_STREAK=1; else unset SABER_NO_STREAK; fi
    SABER_GROUP=$g python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G=$g streak=$st', 'sim_ms=%.2f' % d['roofline']['kernel_ms'], 'traj/s=%.0f' % d['value'])"
  done
done
