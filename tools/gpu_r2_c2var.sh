# C2 (resident kernel): R = 2 ring-depth / tile variants (dev library), ms per 500-step run
for i in 1 2; do
RUNS=3 AW_LIBRARY=tools/ab/libaw_dev.so python tools/run_once.py C2 | tail -1 | sed 's/^/base /'
for v in 1 2 3; do RUNS=3 AW_STREAM_VARIANT=$v AW_LIBRARY=tools/ab/libaw_dev.so python tools/run_once.py C2 | tail -1 | sed "s/^/v$v /"; done
done
