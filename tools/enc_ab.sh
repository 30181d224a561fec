#!/bin/bash
# K1-TC A/B at the full cfg2 size (2048 units x 32K): bench.py's own timing per library, both
# bit widths, libraries alternated twice; optional env per run via ENVS="A=1 B=2;C=3" pairs
for rep in 1 2; do
for l in "$@"; do
  for b in 2 4; do
    PKV_LIB=$PWD/$l timeout 600 python bench.py --steps 5 --warmup 3 --bits $b --no-four-bit --no-cpu --legs none 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$l', 'bits=$b', round(d['value'],1), 'GB/s', round(d['roofline']['frac'],4))"
  done
done
done
