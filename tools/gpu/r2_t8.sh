nvidia-smi -L
for e in 0 1; do GTK_DEFER_EARLY=$e python tools/defer_timeline.py > gpurun_out/t8_tl_early$e.txt 2>&1; done
for rep in 1 2; do
  for e in 0 1; do
    GTK_DEFER_EARLY=$e python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('early=$e', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/t8_ab.txt
  done
done
GTK_DEFER_EARLY=1 python -m pytest tests/test_gpu_recipes.py -x -q -k "defer" 2>&1 | tail -3 > gpurun_out/t8_rec.txt
