#!/bin/bash
# Round-2 profiling pass (one GPU): the bench command's launch list, and one
# ncu --set full capture per headline kernel.  Outputs under gpurun_out/prof2.
set -x
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
# launch list of the bench command (SC headline + streaming), serialised, cold-cache
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_sc.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rows > /dev/null 2>&1
# SC batch screen (k_tc2_screen, Q=65,536 x P=2^20): one launch
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc2_screen -s 1 -c 1 \
  -o $O/sc_batch_screen python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-rows --no-streaming > /dev/null 2>&1
# SC streaming screen (k_tci8_screen, Q=8)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tci8 -s 3 -c 1 \
  -o $O/sc_screen python scripts/sweep_match.py --qs 8 --reps 2 > /dev/null 2>&1
# K1 tracing
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_trace_lane -s 2 -c 1 \
  -o $O/trace_lane env TRACE_ITERS=2 python scripts/trace_probe.py > /dev/null 2>&1
# decision kernel (DS P=10k)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_decision -s 60 -c 3 \
  -o $O/decision env REPS=1 python scripts/ds_probe.py > /dev/null 2>&1
ls -la $O
# SW screen (the SW row) for its DRAM bytes
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tc2_screen -s 2 -c 1 \
  -o $O/sw_screen python scripts/sw_device_probe.py > /dev/null 2>&1 || true
