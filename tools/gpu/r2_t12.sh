nvidia-smi -L
python -m pytest tests/test_gpu_kernels.py -x -q -k "deferred" 2>&1 | tail -3 > gpurun_out/t12_kern.txt
GTK_DEFER_EARLY=1 GTK_FINISH_G=74 python tools/defer_timeline.py > gpurun_out/t12_tl_g74.txt 2>&1
for rep in 1 2; do
  for g in 148 100 74 60; do
    GTK_DEFER_EARLY=1 GTK_FINISH_G=$g python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('early G=$g', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/t12_ab.txt
  done
done
