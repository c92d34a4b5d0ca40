#!/bin/bash
# A/B of alternative engine builds (SABER_LIB) on config 2: tools/lib_ab.sh "libA.so libB.so" [G]
for lib in $1; do
  SABER_GROUP=${2:-32} SABER_LIB=paper_2506_19677_b200/$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib G=${2:-32}', 'sim_ms=%.2f' % d['roofline']['kernel_ms'], 'traj/s=%.0f' % d['value'])"
done
