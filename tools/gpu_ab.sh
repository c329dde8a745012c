# GPU box: full GPU test suite on the in-tree build, then a same-box A/B against build/libaw_old.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 1200 python tools/ab_stream.py --libs new=paper_1906_10811_b200/libaw.so,old=build/libaw_old.so --so ${AB_SO:-2,4,8,12,16} --rounds 2 > gpurun_out/ab.jsonl 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/ab.jsonl
