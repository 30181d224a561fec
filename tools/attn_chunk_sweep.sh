#!/bin/bash
# K3-TC chunking sweep: decode-attention time vs the CTAs-per-SM target (GQA 4 and 7/8 shapes)
for t in ${TARGETS:-4 8 16 32}; do
  for g in 4 8; do
    PKV_ATTN_CTAS_PER_SM=$t timeout 300 python tools/attn_time.py --units 2048 --gqa $g 2>&1 | grep "bits=" | sed "s/^/target=$t gqa=$g /"
  done
  PKV_ATTN_CTAS_PER_SM=$t timeout 300 python tools/attn_time.py --units 112 --tokens 131072 --gqa 7 --bits 2 2>&1 | grep "bits=" | sed "s/^/target=$t cfg3 /"
done
