timeout 900 python -m pytest tests/test_gpu_resident2d.py -x -q > gpurun_out/c1_tests.log 2>&1; echo "rc $?" >> gpurun_out/c1_tests.log
tail -3 gpurun_out/c1_tests.log
python tools/run_once.py C1
ncu --set full --import-source on --clock-control none -k regex:resident2d -c 1 -o gpurun_out/c1_res2d -f python tools/run_once.py C1 > gpurun_out/c1prof.log 2>&1; echo "ncu rc $?"
AW_BENCH_VERBOSE=1 timeout 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
tail -3 gpurun_out/bench_C1.err; cut -c1-300 gpurun_out/bench_C1.json
