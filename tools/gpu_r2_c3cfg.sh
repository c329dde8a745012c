# C3 bench (power-capped, the headline conditions): product R=4 config (16 warps x 2 rows) vs the round-1
# config (8 warps x 4 rows, v7) vs half queue with 4 rows (v6); alternating, 3 rounds
DEV=tools/ab/libaw_dev.so
for i in 1 2 3; do
for arm in prod v7 v6; do
  if [ $arm = prod ]; then timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/c3cfg.json 2>/dev/null
  else AW_LIBRARY=$DEV AW_STREAM_VARIANT=${arm#v} timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/c3cfg.json 2>/dev/null; fi
  python -c "import json; d=json.load(open('gpurun_out/c3cfg.json')); print('$arm', $i, d['value'], d['roofline']['stencil_ms_avg'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
