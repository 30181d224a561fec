#!/bin/bash
# K2 A/B: mining GPU tests on the current build, then tools/mine_bench.py per library
set -x
[ -z "$NO_TEST" ] && timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "mining or kmeans or cfg1 or 32k or mine or verify" 2>&1 | tail -3
for l in "$@"; do
  PKV_LIB=$PWD/$l U=${U:-256} timeout 600 python tools/mine_bench.py 2>&1 | grep "rounds"
done
