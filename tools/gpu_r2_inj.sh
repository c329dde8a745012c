# round 2: streaming kernel with an injection-free instantiation for interior items (smaller unrolled
# loop) -- check, then same-box A/B against the previous build (build/libaw_prev.so@9), so 4..16
timeout 600 python tools/kernel_check.py --R 1,2,3,4,5,6,7,8 --shapes all > gpurun_out/inj_check.log 2>&1; echo "check rc=$?" >> gpurun_out/inj_check.log
tail -2 gpurun_out/inj_check.log
timeout 1500 python tools/ab_stream.py --libs prev=build/libaw_prev.so@9,new=paper_1906_10811_b200/libaw.so --so 4,8,10,12,14,16 --rounds 2 > gpurun_out/ab_inj.jsonl 2>&1
cat gpurun_out/ab_inj.jsonl
timeout 300 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 12 -c 1 \
  -o gpurun_out/stream_inj_so16 -f python tools/ab_stream.py --child 16 --nt 10 > gpurun_out/ncu_inj16.log 2>&1
tail -1 gpurun_out/ncu_inj16.log
