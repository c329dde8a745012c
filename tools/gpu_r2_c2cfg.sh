# round 2: R=2 with 16 consumer warps (RY 2) vs 8 (RY 4): C2 bench (resident on/off) and 512^3 so 4
for lib in base2=build/libaw_base2.so new=paper_1906_10811_b200/libaw.so; do
name=${lib%%=*}; path=${lib#*=}
for r in on off; do
AW_LIBRARY=$path timeout 600 python bench.py --workload C2 --no-cpu-baseline --no-e2e --resident $r > gpurun_out/c2_${name}_$r.json 2> gpurun_out/c2_${name}_$r.err
python -c "import json; d=json.load(open('gpurun_out/c2_${name}_$r.json')); print('C2 $name $r', d['value'], d['ms_per_step'], d['roofline']['stencil_ms_avg'])"
done; done
timeout 600 python tools/ab_stream.py --libs base2=build/libaw_base2.so,new=paper_1906_10811_b200/libaw.so --so 4 --rounds 2 > gpurun_out/ab_c2cfg.jsonl 2>&1
cat gpurun_out/ab_c2cfg.jsonl
timeout 300 python -m pytest tests/test_gpu_resident.py -x -q 2>&1 | tail -1
