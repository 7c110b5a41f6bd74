nvidia-smi -L
for n in 4 2; do
  for c in 1 0; do
    GTK_MERGE_COMPACT=$c python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29560 + n * 2 + c)) bench.py --gpus $n --steps 200 --warmup 20 --no-cpu \
      > gpurun_out/n4b_n${n}_c$c.txt 2>&1
  done
done
