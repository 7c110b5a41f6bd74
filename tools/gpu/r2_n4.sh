# four GPUs: multi-process parity at P=4 and P=3, N=4 / N=2 benches (both modes), N=4 sweep
nvidia-smi -L
python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -8 > gpurun_out/n4_dist.txt
for n in 4 2; do
  for mode in defer plain; do
    GTK_PIPE_MODE=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29530 + n * 2 + ${#mode})) bench.py --gpus $n --steps 200 --warmup 20 \
      > gpurun_out/n4_bench_n${n}_$mode.txt 2>&1
  done
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29549 tools/sweep.py --configs 2,3,4 --no-cpu --protocol --out gpurun_out/r2_sweep_n4.jsonl > gpurun_out/r2_sweep_n4.log 2>&1
