# round 2 (session 3): partial z queues (QJ = 2, 3, 4) for R = 7, 8 -- value checks, then same-box A/B
DEV=tools/ab/libaw_dev.so
for rv in 8:9 8:10 8:11 7:9; do r=${rv%%:*}; v=${rv##*:}
AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R $r --shapes all --nt 24 > gpurun_out/pq_check_${r}_$v.log 2>&1
echo "R=$r v=$v: $(grep -c OK gpurun_out/pq_check_${r}_$v.log) OK, $(grep -c -E 'MISMATCH|ERROR' gpurun_out/pq_check_${r}_$v.log) bad"
done
grep -l -E "MISMATCH|ERROR" gpurun_out/pq_check_*.log && exit 1
timeout 900 python tools/ab_stream.py --libs base=$DEV,v9=$DEV@9,v10=$DEV@10,v11=$DEV@11 --so 16 --rounds 2 > gpurun_out/ab_pq.jsonl 2>&1
timeout 900 python tools/ab_stream.py --libs base=$DEV,v9=$DEV@9 --so 14 --rounds 2 >> gpurun_out/ab_pq.jsonl 2>&1
timeout 900 python tools/ab_stream.py --libs prod=$DEV,old=$DEV@10 --so 12 --rounds 2 >> gpurun_out/ab_pq.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_pq.jsonl'):
    try: d=json.loads(l)
    except: continue
    print(d['lib'], d['round'], d['so'], d['ms_graph'], d['hbm_frac_16B_6537'])"
