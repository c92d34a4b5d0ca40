#!/bin/bash
# One config-2 bench line per environment setting: tools/ab.sh "SABER_ORDER=0" "SABER_ORDER=1" ...
for e in "$@"; do
  env $e python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', 'sim_ms=%.2f' % d['roofline']['kernel_ms'], 'step_ms=%.2f' % d['ms_per_step'], 'traj/s=%.0f' % d['value'])"
done
