# round 2 (session 3): R = 2 half-queue variants on C2, then the full GPU suite + smoke on the final tree
DEV=tools/ab/libaw_dev.so
for v in 4 5; do AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R 2 --shapes all --nt 24 > gpurun_out/c2v_check_$v.log 2>&1; echo "v$v: $(grep -c OK gpurun_out/c2v_check_$v.log) OK $(grep -c -E 'MISMATCH|ERROR' gpurun_out/c2v_check_$v.log) bad"; done
for i in 1 2; do
RUNS=3 python tools/run_once.py C2 | tail -1 | sed 's/^/prod /'
for v in 4 5; do RUNS=3 AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV python tools/run_once.py C2 | tail -1 | sed "s/^/v$v /"; done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
