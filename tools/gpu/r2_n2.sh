# two GPUs: multi-process parity, then the N=2 bench (+ exchange phase trace)
nvidia-smi -L
python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15 > gpurun_out/n2_dist.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 200 --warmup 20 > gpurun_out/n2_bench.txt 2>&1
GTK_TRACE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 50 --warmup 10 > gpurun_out/n2_trace.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --steps 200 --warmup 20 --m 270000 > gpurun_out/n2_bench_r20.txt 2>&1
