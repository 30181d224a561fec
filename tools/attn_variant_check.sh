cp _ab/attn_vfirst.so paper_2510_05176_b200/libpkv_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attn or dist or decode or baseline" 2>&1 | tail -2
cp _ab/attn_cur2.so paper_2510_05176_b200/libpkv_b200.so
NO_TEST=1 UNITS=2048 GQAS="4 8" bash tools/attn_ab.sh _ab/attn_vfirst.so _ab/attn_cur2.so
