# round 2: GPU suite (no full-size), smoke, default bench, C5/C4 quick bench lines
timeout 1200 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench rc $?" >> gpurun_out/bench_C3.err
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_C3.json gpurun_out/bench_C5.json gpurun_out/bench_C2.json; tail -3 gpurun_out/bench_C3.err
