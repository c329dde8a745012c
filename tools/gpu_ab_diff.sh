# GPU box: diffusion parity tests, then a same-box A/B of the diffusion kernel (in-tree build vs build/libaw_old.so)
timeout 900 python -m pytest tests/test_gpu_diffusion.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_diff.log
for r in 0 1; do for lib in new old; do
  if [ $lib = new ]; then L=$PWD/paper_1906_10811_b200/libaw.so; else L=$PWD/build/libaw_old.so; fi
  AW_LIBRARY=$L timeout 600 python tools/bench_diffusion.py --sizes 10000 --orders ${ORD:-2,8,12,16} --nt 300 --reps 2 2>/dev/null | sed "s/^/{\"lib\": \"$lib\", \"round\": $r, \"line\": /; s/\$/}/"
done; done > gpurun_out/ab_diff.jsonl
cat gpurun_out/pytest_diff.log; python - <<'PY'
import json
for l in open("gpurun_out/ab_diff.jsonl"):
    try:
        d = json.loads(l); x = d["line"]
        print(d["lib"], d["round"], x["space_order"], x["kernel_ms_avg"], x["roofline"]["frac"])
    except Exception as e:
        print("?", l[:200])
PY
