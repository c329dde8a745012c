# round 2 (session 3): cluster-resident 2D kernel + stream-ordered ABI trims -- full GPU suite, smoke, C1/C2/C3 lines
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
AW_BENCH_VERBOSE=1 timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
tail -1 gpurun_out/bench_C1.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for w in C1 C2 C3; do python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"; done
