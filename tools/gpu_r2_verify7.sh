# round 2 (session 3): run-begin/end and set_model host trims -- full GPU suite, smoke, C1 line, ncu of the final C4 / C5 kernels
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
AW_BENCH_VERBOSE=1 timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
tail -2 gpurun_out/bench_C1.err; python -c "import json; d=json.load(open('gpurun_out/bench_C1.json')); print('C1', d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'])"
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 30 -c 1 -o gpurun_out/stream_C4_r2b -f \
    python bench.py --workload C4 --steps 1 --warmup 3 --nt 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu C4 rc $?"
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 30 -c 1 -o gpurun_out/stream_C5_r2 -f \
    python bench.py --workload C5 --steps 1 --warmup 3 --nt 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5.log 2>&1; echo "ncu C5 rc $?"
