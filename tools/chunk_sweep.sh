set -x
timeout 600 python -m pytest tests/test_gpu_attn_tc.py -x -q -p no:cacheprovider 2>&1 | tail -2
for c in 32 64 128; do
 for b in 2 4; do
  PKV_TC_CHUNK=$c timeout 600 python bench.py --steps 5 --warmup 3 --bits $b --no-four-bit --no-cpu --legs none 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunk $c bits $b', round(d['value'],1), 'GB/s', round(d['roofline']['frac'],4))"
 done
done
