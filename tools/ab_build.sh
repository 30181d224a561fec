#!/bin/bash
# Build an A/B variant of libpkv_b200.so into _ab/<name>.so with one source replaced:
#   tools/ab_build.sh <name> <source, e.g. pkv_attn> <file.cu to use instead>
# (keep the variant file under _ab/ so its #includes resolve to the current headers), then
# time both on one box: PKV_LIB=$PWD/_ab/<name>.so python bench.py ...
set -e
cd "$(dirname "$0")/.."
python -c "import sys; sys.path.insert(0,'.'); from paper_2510_05176_b200 import build; build.build()"
mkdir -p _ab
B=paper_2510_05176_b200/_build
C=paper_2510_05176_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I$C -Iinclude -c "$3" -o _ab/$1_var.o 2>&1 | grep -i "error" || true
objs=""
for s in pkv_encode pkv_encode_tc pkv_mine pkv_attn pkv_attn_tc pkv_misc pkv_capi; do
  if [ "$s" = "$2" ]; then objs="$objs _ab/$1_var.o"; else objs="$objs $B/$s.o"; fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o _ab/$1.so -lcudart
rm -f _ab/$1_var.o
echo _ab/$1.so
