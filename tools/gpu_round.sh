#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list + full captures of the two hot kernels.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -2 | tee gpurun_out/bench.json
MED="--batch 2 --layers 32 --tokens 32768 --pool 64 --steps 2 --warmup 1 --no-four-bit --no-cpu --e2e-units 8"
if [ -z "$NO_NCU" ]; then
[ -z "$NO_LAUNCH" ] && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-four-bit --no-cpu > /dev/null 2>&1
[ -z "$NO_ENC" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_span -s 3 -c 1 -o gpurun_out/prof_encode -f python bench.py $MED > /dev/null 2>&1
[ -z "$NO_ATTN" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_chunk -s 3 -c 1 -o gpurun_out/prof_attn -f python bench.py $MED > /dev/null 2>&1
fi
ls -la gpurun_out
