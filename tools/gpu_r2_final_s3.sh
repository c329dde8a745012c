# round 2 (session 3): launch list + ncu --set full of the C3 and C4 streaming kernels, then every bench line
python bench.py --steps 1 --warmup 3 --nt 50 --no-cpu-baseline --no-e2e > gpurun_out/plain_C3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_C3_r2.csv \
    python bench.py --steps 1 --warmup 3 --nt 50 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ll.log 2>&1; echo "launch list rc $?"
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 30 -c 1 -o gpurun_out/stream_C3_r2 -f \
    python bench.py --steps 1 --warmup 3 --nt 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo "ncu C3 rc $?"
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 30 -c 1 -o gpurun_out/stream_C4_r2 -f \
    python bench.py --workload C4 --steps 1 --warmup 3 --nt 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu C4 rc $?"
timeout 900 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 1200 python bench.py --workload C5 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
for w in C3 C5 C2 C1; do python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))"; done
