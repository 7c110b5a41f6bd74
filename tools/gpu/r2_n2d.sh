nvidia-smi -L
for n in 2 4; do
  if [ $n = 2 ]; then GS="24 32 40"; else GS="48 64 80 100"; fi
  for g in $GS; do
    GTK_MERGE_COMPACT_CLUSTER=0 GTK_MERGE_COMPACT_G=$g python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29800 + n * 100 + g)) bench.py --gpus $n --steps 200 --warmup 20 --no-cpu \
      2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n G=$g', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/n2d_ab.txt
  done
done
