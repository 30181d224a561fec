#!/bin/bash
# Evidence for profiles/: launch list of the bench command (full cfg2 size) and full ncu
# captures of the three hot kernels at the MED size (batch 2: 512 units x 32K tokens; ncu
# replays each kernel ~40x, so the full-size launch is not captured).  One GPU, never multi-rank.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-four-bit --no-cpu"
MED="python bench.py --batch 2 --layers 32 --tokens 32768 --pool 64 --steps 1 --warmup 3 --no-four-bit --no-cpu --e2e-units 8"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/launches_bench.txt 2>&1
# encode_tc launch 0 is the mining prefill of the pool; launch 1 is the first re-prefill of all units
timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_tc -s 1 -c 1 -o gpurun_out/prof_encode_full -f $MED > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_chunk -s 3 -c 1 -o gpurun_out/prof_attn_full -f $MED > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans -c 1 -o gpurun_out/prof_kmeans -f python bench.py --batch 1 --layers 4 --tokens 32768 --pool 32 --steps 1 --warmup 3 --no-four-bit --no-cpu --e2e-units 8 > /dev/null 2>&1
ls -la gpurun_out
