nvidia-smi -L
for n in 2 4; do
  for cfg in "C=1 G=16" "C=0 G=16" "C=0 G=32" "C=1 G=8" "C=0 G=48"; do
    c=${cfg%% *}; c=${c#C=}; g=${cfg##*G=}
    GTK_MERGE_COMPACT_CLUSTER=$c GTK_MERGE_COMPACT_G=$g python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29700 + n * 10 + g / 8 + c)) bench.py --gpus $n --steps 200 --warmup 20 --no-cpu \
      2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n $cfg', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/n2c_ab.txt
  done
done
