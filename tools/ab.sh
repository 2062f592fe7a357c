#!/bin/bash
# quick A/B numbers for the persistent decode kernel: phase clocks + instruction count / issue
# activity of one launch (ncu), at C2 geometry.  Run under gpurun.
python tools/profile_ws.py "$@" 2>&1 | grep -E "units=|busy|P |C "
ncu --metrics smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum \
    --clock-control none -k regex:decode_ws -s 3 -c 1 python tools/profile_ws.py "$@" 2>&1 | grep -E "inst_executed|issue_active|duration|bank_conflicts|dram__bytes"
