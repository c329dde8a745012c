# round 2: resident kernel, receivers off the critical path -- tests, C2 bench on/off
timeout 240 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/res_tests.log 2>&1; rc=$?; echo "tests rc=$rc" >> gpurun_out/res_tests.log
tail -2 gpurun_out/res_tests.log
if [ $rc != 0 ]; then exit 1; fi
for r in on off; do
timeout 600 python bench.py --workload C2 --no-cpu-baseline --no-e2e --resident $r > gpurun_out/bench_C2_$r.json 2> gpurun_out/bench_C2_$r.err
python -c "import json; d=json.load(open('gpurun_out/bench_C2_$r.json')); print('C2 $r', d['value'], d['ms_per_step'], d['roofline']['stencil_ms_avg'], d['gpu_launches'])"
done
