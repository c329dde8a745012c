# round 2 (session 3): half register queue (HQ) for the high orders -- value checks, then same-box A/B
DEV=tools/ab/libaw_dev.so
for v in 6 7; do
AW_STREAM_VARIANT=$v AW_LIBRARY=$DEV timeout 300 python tools/kernel_check.py --R 6,8 --shapes all --nt 24 > gpurun_out/hq_check_v$v.log 2>&1; echo "check v$v rc=$?" >> gpurun_out/hq_check_v$v.log
tail -12 gpurun_out/hq_check_v$v.log
done
grep -q MISMATCH gpurun_out/hq_check_v*.log && exit 1
timeout 1200 python tools/ab_stream.py --libs base=$DEV,hq8w=$DEV@6,hq12w=$DEV@7 --so 12,16 --rounds 2 > gpurun_out/ab_hq.jsonl 2>&1
cat gpurun_out/ab_hq.jsonl
