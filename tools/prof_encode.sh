# One full ncu capture of the K1-TC encoder at the MED size (tools/gpu_profiles.sh does all kernels)
mkdir -p gpurun_out
MED="python bench.py --batch 2 --layers 32 --tokens 32768 --pool 64 --steps 1 --warmup 3 --no-four-bit --no-cpu --e2e-units 8"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_tc -s 1 -c 1 -o gpurun_out/prof_encode_full -f $MED > gpurun_out/prof_enc.log 2>&1
tail -3 gpurun_out/prof_enc.log
