#!/bin/bash
# GPU-box recipe (gpurun --gpus 4): bench lines at N = 2 and 4, exchange phase
# traces, and tools/sweep.py over BASELINE configs 1-5 at N = 1, 2, 4.
set -u
OUT=gpurun_out/prof_r1_multi
mkdir -p $OUT
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2952$n bench.py --gpus $n > $OUT/bench_n$n.json 2> $OUT/bench_n$n.err
  GTK_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2953$n bench.py --gpus $n --steps 100 --warmup 5 --no-cpu 2>&1 | grep "^\[rank" > $OUT/exchange_trace_n$n.txt
done
GTK_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29523 bench.py --gpus 2 --numel 66000000 --rho 0.01 --precondition 400 --steps 20 --warmup 5 \
    --no-cpu 2>&1 | grep "^\[rank" > $OUT/exchange_trace_n2_k660k.txt
timeout 600 python tools/sweep.py --out $OUT/sweep_n1.jsonl > $OUT/sweep_n1.log 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2954$n tools/sweep.py --configs 2,3,4,5 --out $OUT/sweep_n$n.jsonl > $OUT/sweep_n$n.log 2>&1
done
ls -la $OUT
