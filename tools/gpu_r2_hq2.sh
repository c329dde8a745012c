# round 2 (session 3): HQ variants for R = 4..7 -- value checks, then same-box A/B
DEV=tools/ab/libaw_dev.so
for rv in 4:4 4:5 5:6 5:7 6:9 7:6; do r=${rv%%:*}; v=${rv##*:}
AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R $r --shapes all --nt 24 > gpurun_out/hq2_check_$r_$v.log 2>&1
echo "R=$r v=$v: $(grep -c OK gpurun_out/hq2_check_$r_$v.log) OK, $(grep -c -E 'MISMATCH|ERROR' gpurun_out/hq2_check_$r_$v.log) bad"
done
timeout 900 python tools/ab_stream.py --libs base=$DEV,v4=$DEV@4,v5=$DEV@5 --so 8 --rounds 2 > gpurun_out/ab_hq2.jsonl 2>&1
timeout 900 python tools/ab_stream.py --libs base=$DEV,v6=$DEV@6,v7=$DEV@7 --so 10 --rounds 2 >> gpurun_out/ab_hq2.jsonl 2>&1
timeout 900 python tools/ab_stream.py --libs base=$DEV,v7=$DEV@7,v9=$DEV@9 --so 12 --rounds 2 >> gpurun_out/ab_hq2.jsonl 2>&1
timeout 900 python tools/ab_stream.py --libs base=$DEV,v6=$DEV@6 --so 14 --rounds 2 >> gpurun_out/ab_hq2.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_hq2.jsonl'):
    try: d=json.loads(l)
    except: continue
    print(d['lib'], d['round'], d['so'], d['ms_graph'], d['hbm_frac_16B_6537'])"
