# same-box A/B: round-1 final library vs the current one (per-launch events and graph path)
timeout 900 python tools/ab_stream.py --libs new=paper_1906_10811_b200/libaw.so,r1=build/libaw_r1.so --so 4,8,16 --rounds 2 > gpurun_out/ab_512.jsonl 2>&1
timeout 600 python tools/ab_stream.py --libs new=paper_1906_10811_b200/libaw.so,r1=build/libaw_r1.so --so 4 --rounds 3 --shape 128,128,128 --nt 200 > gpurun_out/ab_128.jsonl 2>&1
cat gpurun_out/ab_512.jsonl gpurun_out/ab_128.jsonl
