#!/bin/bash
# A/B of tensor-core screen builds: SC batch (Q=65,536), SW-size (Q=4,096) and
# the SC streaming i8 screen (Q=8) against P=2^20; plus the SW row shape.
for lib in "$@"; do
  echo "== $lib"
  MOE_LIB=$PWD/$lib timeout 300 python scripts/sweep_match.py --qs 65536,4096,8 --reps 10 2>&1 | grep screen_ms | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['Q'], 'screen_ms %.4f' % d['screen_ms'], 'TOPS %.0f' % d['screen_TOPS'], 'GBps %.0f' % d['screen_GBps'])"
  MOE_LIB=$PWD/$lib timeout 300 python scripts/sweep_match.py --P 10000 --qs 4096 --reps 50 2>&1 | grep screen_ms | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('SW', d['Q'], 'screen_ms %.4f' % d['screen_ms'], 'refine %.4f prep %.4f' % (d['refine_ms'], d['prep_ms']))"
done
