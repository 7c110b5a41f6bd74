nvidia-smi -L
V=$PWD/ab/ft256/libgtopk_b200.so
for rep in 1 2; do
  for g in 60 45 30; do
    for lib in def ft256; do
      if [ $lib = ft256 ]; then export GTK_LIB_PATH=$V; else unset GTK_LIB_PATH; fi
      GTK_FINISH_G=$g python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib G=$g', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/t20_ab.txt
    done
  done
done
unset GTK_LIB_PATH
GTK_LIB_PATH=$V python -m pytest tests/test_gpu_kernels.py -x -q -k "deferred or chained or golden" 2>&1 | tail -3 > gpurun_out/t20_ft256_tests.txt
