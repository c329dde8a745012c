# GPU box: bench lines of every workload at N=1, plus the same-device N=2 functional run of the multi-rank path
for w in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_n1.json 2> gpurun_out/bench_${w}_n1.err
done
AW_BENCH_SAME_DEVICE=1 AW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_n2_same_device.json 2> gpurun_out/bench_n2_same_device.err
for f in gpurun_out/bench_*.json; do echo "== $f"; cut -c1-400 $f; done
