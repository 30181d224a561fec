#!/bin/bash
# Encode-throughput A/B on one box: tools/enc_time.sh lib1.so lib2.so ...  (MED cfg2 shape:
# 512 units x 32K tokens, 2-bit then 4-bit; bench.py's own timing, no extra legs)
for l in "$@"; do
  for b in 2 4; do
    PKV_LIB=$PWD/$l timeout 600 python bench.py --batch 2 --layers 32 --pool 64 --steps 5 --warmup 3 --bits $b \
      --no-four-bit --no-cpu --e2e-pool 8 --legs none 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$l', 'bits=$b', round(d['value'],1), 'GB/s', round(d['roofline']['frac'],4), 'attn', round(d['decode_attn']['ms_per_step'],3))"
  done
done
