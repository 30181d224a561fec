#!/bin/bash
# K3-TC A/B on one box: GPU attention tests on the current build (unless NO_TEST), then
# tools/attn_time.py per library, alternating libraries twice
set -x
[ -z "$NO_TEST" ] && timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attn or dist or decode or baseline" 2>&1 | tail -3
for g in ${GQAS:-4 8}; do
  for rep in 1 2; do
    for l in "$@"; do
      PKV_LIB=$PWD/$l timeout 600 python tools/attn_time.py --units ${UNITS:-512} --gqa $g 2>&1 | tail -2
    done
  done
done
