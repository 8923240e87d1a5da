#!/bin/bash
# A/B of k_trace_lane's L2 run-ahead (MOE_TRACE_PF bytes) at DS, 1,000 and 50 requests.
for R in 1000 50; do
  for pf in 0 32768 65536 131072 262144; do
    echo "R=$R PF=$pf $(TRACE_R=$R TRACE_ITERS=12 MOE_TRACE_PF=$pf python scripts/trace_probe.py | awk '/trace ms/{v[n++]=$3} END{asort(v); print "median_ms", v[int(n/2)]}')"
  done
done
