# C2: upper bound of removing the resident kernel's cross-item waits (wrong results; timing only)
for i in 1 2; do
RUNS=3 python tools/run_once.py C2 | tail -1 | sed 's/^/product /'
RUNS=3 AW_LIBRARY=tools/ab/libaw_dev.so python tools/run_once.py C2 | tail -1 | sed 's/^/dev /'
RUNS=3 AW_RES_NOWAIT=1 AW_LIBRARY=tools/ab/libaw_dev.so python tools/run_once.py C2 | tail -1 | sed 's/^/dev-nowait /'
done
