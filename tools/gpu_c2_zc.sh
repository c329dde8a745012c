# GPU box: C2 (128^3 so 4, L2-resident) bench value vs planes per z chunk (AW_STREAM_ZC; default heuristic = 8)
for zc in default 4 6 8 16; do
  if [ $zc = default ]; then unset AW_STREAM_ZC; else export AW_STREAM_ZC=$zc; fi
  timeout 300 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$zc', d['value'], d['roofline']['stencil_ms_avg'])"
done
