timeout 900 python -m pytest tests/test_gpu_resident2d.py -x -q 2>&1 | tail -2
python tools/c1_sparse_cost.py
timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
python -c "import json; d=json.load(open('gpurun_out/bench_C1.json')); print('C1', d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'])"
