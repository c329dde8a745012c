# round 2: boundary-first team signalling -- team tests (virtual ranks, cudaIpc processes), same-device N=2 bench
timeout 900 python -m pytest tests -m gpu -x -q -k "team" > gpurun_out/team_tests.log 2>&1; rc=$?; echo "team rc=$rc" >> gpurun_out/team_tests.log
tail -3 gpurun_out/team_tests.log
if [ $rc != 0 ]; then exit 1; fi
AW_BENCH_SAME_DEVICE=1 AW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --no-cpu-baseline --no-e2e --workload C5 > gpurun_out/bench_n2_same.json 2> gpurun_out/bench_n2_same.err; echo "n2 rc $?" >> gpurun_out/bench_n2_same.err
tail -2 gpurun_out/bench_n2_same.err; cat gpurun_out/bench_n2_same.json
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
