# round 2: high-order kernel with the streams loaded one output plane ahead (AW_H_PREFETCH=1) --
# check, A/B against the generic streaming kernel (AW_STREAM_VARIANT=9), ncu of so 16
DEV=build/libaw_dev.so
AW_LIBRARY=$DEV timeout 900 python tools/kernel_check.py --R 5,6,7,8 --shapes all > gpurun_out/h_check.log 2>&1; echo "check rc=$?" >> gpurun_out/h_check.log
tail -2 gpurun_out/h_check.log
timeout 1200 python tools/ab_stream.py --libs old=$DEV@9,new=$DEV --so 10,12,14,16 --rounds 2 > gpurun_out/ab_h2.jsonl 2>&1
cat gpurun_out/ab_h2.jsonl
AW_LIBRARY=$DEV timeout 600 ncu --set full --import-source on --clock-control none -k regex:hstream_kernel --launch-skip 12 -c 1 \
  -o gpurun_out/hstream6_so16 -f python tools/ab_stream.py --child 16 --nt 10 > gpurun_out/ncu_h16.log 2>&1
tail -1 gpurun_out/ncu_h16.log
