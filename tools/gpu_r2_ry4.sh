# round 2 (session 3): half queue with 4 rows per thread (8 consumer warps, 64 x 32 tiles), R = 4..8
DEV=tools/ab/libaw_dev.so
for rv in 4:6 5:8 6:15 6:16 7:12 8:12 8:13; do r=${rv%%:*}; v=${rv##*:}
AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R $r --shapes all --nt 24 > gpurun_out/ry4_check_${r}_$v.log 2>&1
echo "R=$r v=$v: $(grep -c OK gpurun_out/ry4_check_${r}_$v.log) OK, $(grep -c -E 'MISMATCH|ERROR' gpurun_out/ry4_check_${r}_$v.log) bad"
done
timeout 600 python tools/ab_stream.py --libs prod=$DEV,v6=$DEV@6 --so 8 --rounds 2 > gpurun_out/ab_ry4.jsonl 2>&1
timeout 600 python tools/ab_stream.py --libs prod=$DEV,v8=$DEV@8 --so 10 --rounds 2 >> gpurun_out/ab_ry4.jsonl 2>&1
timeout 600 python tools/ab_stream.py --libs v14=$DEV@14,v15=$DEV@15,v16=$DEV@16 --so 12 --rounds 2 >> gpurun_out/ab_ry4.jsonl 2>&1
timeout 600 python tools/ab_stream.py --libs prod=$DEV,v12=$DEV@12 --so 14 --rounds 2 >> gpurun_out/ab_ry4.jsonl 2>&1
timeout 600 python tools/ab_stream.py --libs prod=$DEV,v12=$DEV@12,v13=$DEV@13 --so 16 --rounds 2 >> gpurun_out/ab_ry4.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_ry4.jsonl'):
    try: d=json.loads(l)
    except: continue
    print(d['lib'], d['round'], d['so'], d['ms_graph'], d['hbm_frac_16B_6537'])"
