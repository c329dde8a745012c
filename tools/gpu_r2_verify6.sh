# round 2 (session 3): half queue + 4 rows per thread for R = 6..8 -- full GPU suite, smoke, C4 / C5 lines, N=2 same-device C5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 1200 python bench.py --workload C5 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
for w in C4 C5; do python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['stencil_ms_avg'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
AW_BENCH_SAME_DEVICE=1 AW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --no-cpu-baseline --no-e2e --workload C5 > gpurun_out/bench_n2_same.json 2> gpurun_out/bench_n2_same.err; echo "n2 rc $?"
cut -c1-300 gpurun_out/bench_n2_same.json
timeout 1200 python -m tests.parity_full --cases C5,C4g --out gpurun_out/parity_s3.jsonl > gpurun_out/parity_s3.log 2>&1; echo "parity rc $?"; cut -c1-330 gpurun_out/parity_s3.jsonl
