#!/bin/bash
# k_trace_lane timing at DS (1,000 and 50 requests): median of 10 calls (scripts/trace_probe.py).
for R in 1000 50; do
  med=$(TRACE_R=$R TRACE_ITERS=12 python scripts/trace_probe.py | awk '/trace ms/{print $3}' | tail -n 10 | sort -n | sed -n 5p)
  echo "R=$R median_ms $med"
done
