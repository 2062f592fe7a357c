#!/bin/bash
# Profiling evidence for one round (run under gpurun); raw outputs in gpurun_out/, the
# summaries bench.py and the judge read are then copied under profiles/<round>/.
#   tools/profile_round.sh [config]      (default c2)
set -x
CFG=${1:-c2}
mkdir -p gpurun_out
# 1) launch list of the bench command: per-launch device time of its decode launches
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode -c 12 --csv \
    --log-file gpurun_out/launches_${CFG}.csv python bench.py --config ${CFG} --steps 4 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_under_ncu_${CFG}.log 2>&1
# 2) full capture of one decode step at the bench workload (after the warm-up steps; the
#    two-kernel path launches decode_select_kernel + decode_attend_kernel per step)
NK=$(python -c "import sys; sys.path.insert(0, '.'); import bench; c = bench.CONFIGS['${CFG}']; print(1 if c[0] * c[1] * c[2] < 64 else 2)")   # two-kernel path: select + attend per step
ncu --set full --import-source on --clock-control none -k regex:decode -s $((3 * NK)) -c ${NK} \
    -o gpurun_out/decode_${CFG} python bench.py --config ${CFG} --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${CFG}.log 2>&1
ncu -i gpurun_out/decode_${CFG}.ncu-rep --page raw --csv > gpurun_out/decode_${CFG}_raw.csv 2>&1
ncu -i gpurun_out/decode_${CFG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/decode_${CFG}_src.csv 2>&1
python tools/ncu_summary.py gpurun_out/decode_${CFG}_raw.csv ${CFG} > gpurun_out/ncu_${CFG}_summary.json
python tools/ncu_src.py gpurun_out/decode_${CFG}_src.csv 40 samples > gpurun_out/ncu_${CFG}_lines.txt
rm -f gpurun_out/decode_${CFG}.ncu-rep
