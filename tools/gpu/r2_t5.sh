nvidia-smi -L
python -m pytest tests/test_gpu_kernels.py -x -q -k "deferred or chained" 2>&1 | tail -15 > gpurun_out/t5_kern.txt
python -m pytest tests/test_gpu_recipes.py -x -q 2>&1 | tail -15 > gpurun_out/t5_recipes.txt
for rep in 1 2; do
  for mode in defer plain chain; do
    GTK_PIPE_MODE=$mode python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', d['value'], d['roofline']['launch_ms'], d['kernels_per_step'], d['stages_ms'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/t5_ab.txt
  done
done
