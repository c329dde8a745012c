# round 2: high-order kernel (aw_hstream.cuh) -- correctness (stream vs v1 for R=5..8, the GPU suite),
# same-box A/B against the generic streaming kernel (AW_STREAM_VARIANT=9), ncu of so 16
DEV=build/libaw_dev.so
timeout 900 python tools/kernel_check.py --R 5,6,7,8 --shapes all > gpurun_out/h_check.log 2>&1; echo "check rc=$?" >> gpurun_out/h_check.log
tail -3 gpurun_out/h_check.log
timeout 1200 python tools/ab_stream.py --libs old=$DEV@9,new=$DEV --so 10,12,14,16 --rounds 2 > gpurun_out/ab_h.jsonl 2>&1
cat gpurun_out/ab_h.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hstream_kernel --launch-skip 12 -c 1 \
  -o gpurun_out/hstream_so16 -f python tools/ab_stream.py --child 16 --nt 10 > gpurun_out/ncu_h16.log 2>&1
tail -2 gpurun_out/ncu_h16.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
