#!/bin/bash
# Profiling evidence for one round (run under gpurun); outputs in gpurun_out/
set -x
mkdir -p gpurun_out
# 1) launch list of the bench command (decode kernels only), per-launch device time
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode -c 20 --csv \
    --log-file gpurun_out/launches_c2.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
# 2) full capture of the hot kernel at the bench workload (C2, all 4096 units)
ncu --set full --import-source on --clock-control none -k regex:decode_ws -c 1 \
    -o gpurun_out/decode_ws_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/decode_ws_c2.ncu-rep --page raw --csv > gpurun_out/decode_ws_c2_raw.csv 2>&1
ncu -i gpurun_out/decode_ws_c2.ncu-rep --page details --csv > gpurun_out/decode_ws_c2_details.csv 2>&1
