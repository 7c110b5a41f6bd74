# two GPUs: multi-process parity (deferred + plain pipelines), N=2 bench both modes, trace
nvidia-smi -L
python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15 > gpurun_out/n2b_dist.txt
for mode in defer plain; do
  GTK_PIPE_MODE=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 2952$([ $mode = defer ] && echo 1 || echo 2) bench.py --gpus 2 --steps 200 --warmup 20 \
    > gpurun_out/n2b_bench_$mode.txt 2>&1
done
GTK_PIPE_MODE=defer python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29525 tools/sweep.py --configs 2,3,4 --no-cpu --protocol --out gpurun_out/r2_sweep_n2.jsonl > gpurun_out/r2_sweep_n2.log 2>&1
