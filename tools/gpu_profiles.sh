#!/bin/bash
# Evidence for profiles/: launch list of the bench command and full captures of the
# two hot kernels at the bench configuration (one GPU, never multi-rank).
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-four-bit --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_span -s 3 -c 1 -o gpurun_out/prof_encode_full -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_chunk -s 3 -c 1 -o gpurun_out/prof_attn_full -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans -c 1 -o gpurun_out/prof_kmeans -f python bench.py --batch 1 --layers 4 --tokens 32768 --pool 32 --steps 1 --warmup 3 --no-four-bit --no-cpu --e2e-units 8 > /dev/null 2>&1
ls -la gpurun_out
