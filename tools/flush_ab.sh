for l in paper_2510_05176_b200/libpkv_b200.so _ab/enc_old.so; do
PKV_LIB=$PWD/$l timeout 1200 python bench.py --steps 3 --warmup 3 --no-four-bit --no-cpu --legs cfg4 --batch 1 2>&1 | tail -1 > gpurun_out/fl.json
python -c "
import json; d=json.load(open('gpurun_out/fl.json')); c4=d['cfg4']
print('$l', 'late tok/s', round(c4['late_tokens_per_s']), 'flush ms', c4.get('late_flush_ms'), 'P', c4['late_patterns'])"
done
