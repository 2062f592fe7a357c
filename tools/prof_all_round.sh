# Every profiling artefact of the round in one gpurun call; copy gpurun_out/r2b/* and the
# summaries to profiles/<round>/ afterwards.  Bench lines at 50 steps (the 300-step default
# runs into the board power cap: C2 0.867 vs 0.837 ms).
set -x
mkdir -p gpurun_out/r2b
for c in c2 c3 c4 c5; do python bench.py --config $c --steps 50 > gpurun_out/r2b/bench_$c.json 2> gpurun_out/r2b/bench_$c.err; done
python bench.py --policy per-head --config c4 --steps 50 > gpurun_out/r2b/bench_c4_perhead.json 2>/dev/null
for c in c2 c3 c4; do bash tools/profile_round.sh $c; done
# compute-sanitizer is closed on the GPU pool since late round 2 (the committed
# profiles/round2/sanitize_*.log are from before); run tools/sanitize_all.sh where it is allowed
python tools/sass_opcodes.py > gpurun_out/r2b/sass_opcodes.txt
for c in c2 c4 c3; do python tools/exchange_cost.py $c 8; done > gpurun_out/r2b/exchange_cost.txt
python tools/bench_perhead.py --tokens 4096 32768 > gpurun_out/r2b/perhead_api_bench.jsonl
ls gpurun_out
