# round 2 (session 3): R = 6 half-queue variants (ring depths, 3 / 4 rows per thread) -- checks, A/B at so 12
DEV=tools/ab/libaw_dev.so
for v in 11 12 13 14; do
AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R 6 --shapes all --nt 24 > gpurun_out/r6v_check_$v.log 2>&1
echo "v=$v: $(grep -c OK gpurun_out/r6v_check_$v.log) OK, $(grep -c -E 'MISMATCH|ERROR' gpurun_out/r6v_check_$v.log) bad"
done
timeout 1200 python tools/ab_stream.py --libs prod=$DEV,v11=$DEV@11,v12=$DEV@12,v13=$DEV@13,v14=$DEV@14 --so 12 --rounds 2 > gpurun_out/ab_r6v.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_r6v.jsonl'):
    try: d=json.loads(l)
    except: continue
    print(d['lib'], d['round'], d['so'], d['ms_graph'], d['hbm_frac_16B_6537'])"
