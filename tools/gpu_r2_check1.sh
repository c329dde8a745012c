# round 2, first GPU call: full GPU suite (without the full-size cases), the full-size parity report, host info
nproc > gpurun_out/host.txt; lscpu >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt; which numactl >> gpurun_out/host.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 1500 python -m tests.parity_full --out gpurun_out/parity_full.jsonl > gpurun_out/parity_full.log 2>&1; echo "parity rc $?" >> gpurun_out/parity_full.log
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/parity_full.jsonl
