for i in 1 2; do
RUNS=6 python tools/run_once.py C1 | tail -2 | sed 's/^/t1024 /'
RUNS=6 AW_LIBRARY=tools/ab/libaw_r2t512.so python tools/run_once.py C1 | tail -2 | sed 's/^/t512 /'
RUNS=6 AW_LIBRARY=tools/ab/libaw_r2t256.so python tools/run_once.py C1 | tail -2 | sed 's/^/t256 /'
done
