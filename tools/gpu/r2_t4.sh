nvidia-smi -L
python -m pytest tests/test_gpu_kernels.py -x -q -k "chained" 2>&1 | tail -5 > gpurun_out/t4_chain.txt
for rep in 1 2; do
  for chain in 0 1; do
    GTK_PIPE_CHAIN=$chain python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chain=$chain', d['value'], d['roofline']['launch_ms'], d['kernels_per_step'], d['stages_ms'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/t4_ab.txt
  done
done
