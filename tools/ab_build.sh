#!/bin/bash
# Build an A/B variant of libpkv_b200.so into _ab/<name>.so with one source replaced:
#   tools/ab_build.sh <name> <file.cu to use as pkv_encode_tc.cu>
# then time both on one box: PKV_LIB=$PWD/_ab/<name>.so python bench.py ...
set -e
cd "$(dirname "$0")/.."
python -c "import sys; sys.path.insert(0,'.'); from paper_2510_05176_b200 import build; build.build()"
mkdir -p _ab
B=paper_2510_05176_b200/_build
C=paper_2510_05176_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I$C -Iinclude -c "$2" -o _ab/$1_tc.o 2>&1 | grep -v "TWO_M15\|^ *\^\|^$\|declared but never" || true
objs=""
for s in pkv_encode pkv_mine pkv_attn pkv_misc pkv_capi; do objs="$objs $B/$s.o"; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs _ab/$1_tc.o -o _ab/$1.so -lcudart
echo _ab/$1.so
