#!/bin/bash
# K2 per-CTA phase timing of a printf-instrumented build (first pass / seeding / Lloyd per unit-side)
for l in "$@"; do echo == $l; PKV_LIB=$PWD/$l U=256 REPS=1 timeout 600 python tools/mine_bench.py > gpurun_out/mine_phase.txt 2>&1; grep -c CTA gpurun_out/mine_phase.txt; done
