# round 2: 16 consumer warps (RY 2) for R = 1..4 vs the 8-warp (RY 4) build base2: 512^3 so 2/4/6/8, C3 bench
timeout 900 python tools/ab_stream.py --libs base2=build/libaw_base2.so,new=paper_1906_10811_b200/libaw.so --so 2,4,6,8 --rounds 2 > gpurun_out/ab_rycfg.jsonl 2>&1
cat gpurun_out/ab_rycfg.jsonl
timeout 600 python tools/kernel_check.py --R 1,2,3,4 --shapes all > gpurun_out/ry_check.log 2>&1; echo "check rc=$?" >> gpurun_out/ry_check.log; tail -1 gpurun_out/ry_check.log
