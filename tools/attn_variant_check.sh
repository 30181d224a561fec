#!/bin/bash
# K3-TC variant check: GPU attention tests with the variant library in place, then the A/B timing
#   bash tools/attn_variant_check.sh _ab/<variant>.so _ab/<baseline>.so
cp "$1" paper_2510_05176_b200/libpkv_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attn or dist or decode or baseline" 2>&1 | tail -2
cp "$2" paper_2510_05176_b200/libpkv_b200.so
NO_TEST=1 UNITS=2048 GQAS="4 8" bash tools/attn_ab.sh "$1" "$2"
