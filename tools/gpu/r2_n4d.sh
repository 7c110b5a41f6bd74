nvidia-smi -L
python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3 > gpurun_out/n4d_dist.txt
for n in 2 4; do
  for c in 0 1; do
    GTK_MERGE_COMPACT_COOP=$c python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29920 + n * 2 + c)) \
      bench.py --gpus $n --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n coop=$c', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/n4d_ab.txt
  done
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29931 tools/defer_timeline.py > gpurun_out/n4d_tl_n2.txt 2>&1
