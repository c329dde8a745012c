# GPU box, end of round: GPU tests, smoke, bench lines (C3 default, C4, C5 at N=1), ncu launch list and one
# `ncu --set full` capture of the streaming kernel on C3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for w in C4 C5; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_${w}_n1.json 2> gpurun_out/bench_${w}_n1.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:aw:: -c 400 --csv \
  --log-file gpurun_out/launches_C3_nt50.csv python bench.py --steps 1 --warmup 3 --nt 50 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 25 -c 1 -f \
  -o gpurun_out/stream_kernel_C3 python bench.py --steps 1 --warmup 3 --nt 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -2 gpurun_out/ncu_full.log; cut -c1-300 gpurun_out/bench_C3.json
