# GPU box: correctness of AW_STREAM_VARIANT=$V for R = 6, 8 (streaming vs v1 kernel, value-identical),
# then a same-box A/B of the default configuration vs the variant at so 12 / 16
V=${V:-4}
AW_STREAM_VARIANT=$V timeout 600 python tools/kernel_check.py --R ${VR:-6,8} --shapes all > gpurun_out/variant_check.log 2>&1; echo "check rc=$?" >> gpurun_out/variant_check.log
timeout 900 python tools/ab_stream.py --libs base=paper_1906_10811_b200/libaw.so,v$V=paper_1906_10811_b200/libaw.so@$V --so ${AB_SO:-12,16} --rounds 2 > gpurun_out/ab_variant.jsonl 2>&1
tail -4 gpurun_out/variant_check.log; cat gpurun_out/ab_variant.jsonl
