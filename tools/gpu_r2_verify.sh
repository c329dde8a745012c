# round 2: verify the product build (GPU suite, smoke, default bench)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench rc $?" >> gpurun_out/bench_C3.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_C3.json; tail -2 gpurun_out/bench_C3.err
