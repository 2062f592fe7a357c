set -x
mkdir -p gpurun_out/r2b
for c in c2 c3 c4 c5; do python bench.py --config $c > gpurun_out/r2b/bench_$c.json 2> gpurun_out/r2b/bench_$c.err; done
python bench.py --policy per-head --config c4 > gpurun_out/r2b/bench_c4_perhead.json 2>/dev/null
for c in c2 c3 c4; do bash tools/profile_round.sh $c; done
timeout 1500 bash tools/sanitize_all.sh
python tools/sass_opcodes.py > gpurun_out/r2b/sass_opcodes.txt
ls gpurun_out
