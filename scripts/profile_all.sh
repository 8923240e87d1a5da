set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof/launches_sw.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-rows --no-batch > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tc2_screen -s 3 -c 1 -o gpurun_out/prof/sw_screen python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rows --no-streaming > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_prep_u8|k_refine" -s 4 -c 2 -o gpurun_out/prof/sw_prep_refine python scripts/sw_device_probe.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tci8 -s 3 -c 1 -o gpurun_out/prof/sc_screen python scripts/sweep_match.py --qs 8 --reps 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_trace_u8|k_trace_commit" -s 2 -c 2 -o gpurun_out/prof/trace python scripts/trace_probe.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_replay_block|k_apply_block" -s 2 -c 2 -o gpurun_out/prof/replay env NL_STEPS=3000 python scripts/nl_probe.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_dec_dist|k_order|k_member" -s 90 -c 6 -o gpurun_out/prof/decide env REPS=1 python scripts/ds_probe.py > /dev/null 2>&1
ls -la gpurun_out/prof
