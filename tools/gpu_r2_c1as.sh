# C1: st.async neighbour sync vs cluster barrier -- parity tests, then timing (ms per 100-step run)
timeout 300 python tools/run_once.py C1 || exit 1
timeout 900 python -m pytest tests/test_gpu_resident2d.py -x -q 2>&1 | tail -2
for i in 1 2; do
RUNS=6 python tools/run_once.py C1 | tail -1 | sed 's/^/async /'
RUNS=6 AW_R2_SYNC=cluster AW_LIBRARY=tools/ab/libaw_dev.so python tools/run_once.py C1 | tail -1 | sed 's/^/cluster /'
done
timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
python -c "import json; d=json.load(open('gpurun_out/bench_C1.json')); print('C1', d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'])"
