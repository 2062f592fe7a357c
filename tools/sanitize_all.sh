#!/bin/bash
# compute-sanitizer over tools/sanitize_decode.py (run under gpurun); logs to gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_decode.py 300 4096 \
    > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}.log
done
# the per-head float64 kernels (lut / score / top-k / attend)
for tool in memcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_perhead.py \
    > gpurun_out/sanitize_perhead_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_perhead_${tool}.log
done
