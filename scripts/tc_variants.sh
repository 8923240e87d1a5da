#!/bin/bash
# A/B of tensor-core screen builds: SC batch (Q=65,536) and SW-size (Q=4,096) screens.
for lib in "$@"; do
  echo "== $lib"
  MOE_LIB=$PWD/$lib timeout 300 python scripts/sweep_match.py --qs 65536,4096 --reps 10 2>&1 | grep screen_ms | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['Q'], 'screen_ms %.3f' % d['screen_ms'], 'TOPS %.0f' % d['screen_TOPS'])"
done
