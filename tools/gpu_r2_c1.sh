# round 2: one-CTA resident 2D kernel (C1) -- parity tests, C1 bench line, per-call host breakdown
timeout 900 python -m pytest tests/test_gpu_resident2d.py tests/test_gpu_2d.py -x -q > gpurun_out/c1_tests.log 2>&1; echo "rc $?" >> gpurun_out/c1_tests.log
tail -5 gpurun_out/c1_tests.log
timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
cat gpurun_out/bench_C1.json; tail -3 gpurun_out/bench_C1.err
AW_BENCH_VERBOSE=1 timeout 600 python bench.py --workload C1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C1_verbose.json 2> gpurun_out/bench_C1_verbose.err
tail -12 gpurun_out/bench_C1_verbose.err
timeout 600 python bench.py --workload C1 --resident off --no-cpu-baseline > gpurun_out/bench_C1_off.json 2> gpurun_out/bench_C1_off.err
cat gpurun_out/bench_C1_off.json
