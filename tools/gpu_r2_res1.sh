# round 2: resident multi-step kernel (small grids) -- hang guard, parity tests, C2/C1 bench lines
timeout 180 python -m pytest tests/test_gpu_resident.py -x -q -k "test_resident_matches_oracle and resident-shape0" > gpurun_out/res_quick.log 2>&1; rc=$?; echo "quick rc=$rc" >> gpurun_out/res_quick.log
tail -3 gpurun_out/res_quick.log
if [ $rc != 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/res_tests.log
tail -3 gpurun_out/res_tests.log
timeout 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench rc $?" >> gpurun_out/bench_C2.err
python -c "import json; d=json.load(open('gpurun_out/bench_C2.json')); print('C2', d['value'], d['ms_per_step'], d['roofline']['stencil_ms_avg'], d['e2e']['value'], d['gpu_launches'])"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
