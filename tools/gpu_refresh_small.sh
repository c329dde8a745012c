# GPU box: bench lines of the small configurations (C1, C2), the paper's diffusion benchmark, and the
# same-device N=2 functional run of the multi-rank bench path
for w in C1 C2; do timeout 600 python bench.py --workload $w > gpurun_out/bench_${w}_n1.json 2> gpurun_out/bench_${w}_n1.err; done
timeout 900 python tools/bench_diffusion.py --sizes 2500,10000 --orders 2,4,8,12,16 > gpurun_out/diffusion_next2.jsonl 2> gpurun_out/diffusion.err
AW_BENCH_SAME_DEVICE=1 AW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_n2_same_device.json 2> gpurun_out/bench_n2_same_device.err
for f in gpurun_out/bench_C1_n1.json gpurun_out/bench_C2_n1.json gpurun_out/bench_n2_same_device.json; do cut -c1-250 $f; done
cut -c1-200 gpurun_out/diffusion_next2.jsonl
