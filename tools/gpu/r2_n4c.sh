nvidia-smi -L
python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3 > gpurun_out/n4c_dist.txt
python -m pytest tests/test_gpu_exchange_loopback.py -x -q 2>&1 | tail -3 >> gpurun_out/n4c_dist.txt
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900 + n)) \
    bench.py --gpus $n --steps 200 --warmup 20 > gpurun_out/n4c_bench_n$n.txt 2>&1
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 tools/defer_timeline.py > gpurun_out/n4c_tl_n2.txt 2>&1
