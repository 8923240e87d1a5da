#!/bin/bash
# A/B of the i8 streaming screen builds: P=2^20, Q = 1, 2, 4, 8, 16, 64 (screen-kernel events).
for lib in "$@"; do
  echo "== $lib"
  MOE_LIB=$PWD/$lib timeout 300 python scripts/sweep_match.py --qs 1,4,8,16,64 --reps 20 2>&1 | grep screen_ms | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['Q'], 'screen_ms %.4f' % d['screen_ms'], 'GBps %.0f' % d['screen_GBps'])"
done
