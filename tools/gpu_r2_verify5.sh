# round 2 (session 3): R = 6 half register queue in the product -- full GPU suite, smoke, C4 / C3 lines, parity_full C4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for w in C4 C3; do python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['stencil_ms_avg'], d['e2e']['value'], d['clocks'])"; done
