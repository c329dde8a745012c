# round 2: warpgroup-layout (setmaxnreg, 12 consumer warps) variants of R = 6, 8 -- correctness vs the v1
# kernel, same-box A/B against the product configuration, and a source-level ncu capture of so 16
DEV=build/libaw_dev.so
for V in 4 5; do
  AW_LIBRARY=$DEV AW_STREAM_VARIANT=$V timeout 600 python tools/kernel_check.py --R 6,8 --shapes all > gpurun_out/wg_check_v$V.log 2>&1; echo "check rc=$?" >> gpurun_out/wg_check_v$V.log
done
timeout 1200 python tools/ab_stream.py --libs base=paper_1906_10811_b200/libaw.so,v4=$DEV@4,v5=$DEV@5 --so 12,16 --rounds 2 > gpurun_out/ab_wg.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 12 -c 1 \
  -o gpurun_out/stream_so16_base -f python tools/ab_stream.py --child 16 --nt 10 > gpurun_out/ncu_base.log 2>&1
AW_LIBRARY=$DEV AW_STREAM_VARIANT=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 12 -c 1 \
  -o gpurun_out/stream_so16_v4 -f python tools/ab_stream.py --child 16 --nt 10 > gpurun_out/ncu_v4.log 2>&1
tail -2 gpurun_out/wg_check_v*.log; cat gpurun_out/ab_wg.jsonl; tail -2 gpurun_out/ncu_base.log gpurun_out/ncu_v4.log
