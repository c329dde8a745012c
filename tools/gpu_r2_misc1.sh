timeout 600 python -m pytest tests/test_gpu_boundary.py -x -q > gpurun_out/boundary.log 2>&1; echo "rc $?" >> gpurun_out/boundary.log; tail -3 gpurun_out/boundary.log
timeout 1200 python -m tests.parity_full --cases C4g --out gpurun_out/parity_C4g.jsonl > gpurun_out/parity_C4g.log 2>&1; echo "parity rc $?"; cat gpurun_out/parity_C4g.jsonl
