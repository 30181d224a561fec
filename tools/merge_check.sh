#!/bin/bash
# attention merge-kernel variant: GPU attention tests, then decode-attention timing per library
cp "$1" paper_2510_05176_b200/libpkv_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attn or dist or decode or baseline or parity or edges or snapshot" 2>&1 | tail -2
NO_TEST=1 UNITS=2048 GQAS="4 8" bash tools/attn_ab.sh "$1" "$2"
