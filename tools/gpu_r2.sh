#!/bin/bash
# Round-2 GPU session: parity tests, smoke, bench (all legs), launch list, full ncu captures of
# the three hot kernels (skipping warm-up launches), compute-sanitizer on the smoke path.
# One GPU, never multi-rank under ncu.  Outputs under gpurun_out/ (scratch; summaries -> profiles/).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
if [ -z "$NO_TEST" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_gputest.txt 2>&1
tail -15 gpurun_out/${TAG}_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
fi
if [ -z "$NO_BENCH" ]; then
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
cat gpurun_out/${TAG}_bench.json | head -c 3000; echo
fi
if [ -z "$NO_NCU" ]; then
B="python bench.py --steps 2 --warmup 3 --no-four-bit --no-cpu --legs none"
MED="python bench.py --batch 2 --layers 32 --tokens 32768 --pool 64 --steps 1 --warmup 3 --no-four-bit --no-cpu --e2e-pool 8 --legs none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_tc -s 2 -c 1 -o gpurun_out/${TAG}_prof_encode -f $MED > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/${TAG}_prof_attn -f $MED > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans -s 1 -c 1 -o gpurun_out/${TAG}_prof_kmeans -f python bench.py --batch 1 --layers 4 --tokens 32768 --pool 32 --steps 1 --warmup 3 --no-four-bit --no-cpu --e2e-pool 8 --legs none > /dev/null 2>&1
fi
if [ -z "$NO_SAN" ]; then
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_san_smoke_$t.txt 2>&1
  tail -3 gpurun_out/${TAG}_san_smoke_$t.txt
done
fi
ls -la gpurun_out
