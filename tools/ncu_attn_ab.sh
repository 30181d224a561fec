for l in paper_2510_05176_b200/libpkv_b200.so _ab/attn_old.so; do
 n=$(basename $l .so)
 PKV_LIB=$PWD/$l timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 5 -c 1 -o gpurun_out/ab_$n -f python tools/attn_time.py --units 512 --gqa 4 --bits 2 > /dev/null 2>&1
done
ls gpurun_out
