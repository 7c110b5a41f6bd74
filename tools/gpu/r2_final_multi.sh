# four GPUs: the multi-GPU suite, N = 2 / 4 bench lines (default deferred and the
# non-deferred step), sweeps with the reference-protocol rows, N = 2 timeline
nvidia-smi -L
OUT=${OUT:-gpurun_out/final_multi}
mkdir -p $OUT
python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3 > $OUT/dist.txt
for n in 2 4; do
  for mode in defer plain; do
    GTK_PIPE_MODE=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29970 + n * 2 + ${#mode} % 2)) bench.py --gpus $n --steps 200 --warmup 20 > $OUT/bench_n${n}_$mode.json 2> $OUT/bench_n${n}_$mode.err
  done
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29990 + n)) \
    tools/sweep.py --configs 2,3,4,5 --no-cpu --protocol --out $OUT/sweep_n$n.jsonl > $OUT/sweep_n$n.log 2>&1
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29999 \
  tools/defer_timeline.py > $OUT/timeline_n2.txt 2>&1
ls -la $OUT
