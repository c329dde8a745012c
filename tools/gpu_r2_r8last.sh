DEV=tools/ab/libaw_dev.so
for rv in 8:15 8:16 7:13; do r=${rv%%:*}; v=${rv##*:}
AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R $r --shapes all --nt 24 > gpurun_out/r8l_check_${r}_$v.log 2>&1
echo "R=$r v=$v: $(grep -c OK gpurun_out/r8l_check_${r}_$v.log) OK, $(grep -c -E 'MISMATCH|ERROR' gpurun_out/r8l_check_${r}_$v.log) bad"
done
timeout 600 python tools/ab_stream.py --libs prod=$DEV,v15=$DEV@15,v16=$DEV@16 --so 16 --rounds 2 > gpurun_out/ab_r8l.jsonl 2>&1
timeout 600 python tools/ab_stream.py --libs prod=$DEV,v13=$DEV@13 --so 14 --rounds 2 >> gpurun_out/ab_r8l.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_r8l.jsonl'):
    try: d=json.loads(l)
    except: continue
    print(d['lib'], d['round'], d['so'], d['ms_graph'], d['hbm_frac_16B_6537'])"
