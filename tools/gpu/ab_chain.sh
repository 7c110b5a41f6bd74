# A/B on one B200: main-pass register cap (min blocks 3 vs 1) x chained select on/off
set -x
nvidia-smi -L
for rep in 1 2; do
for lib in default v1; do
  for chain in 1 0; do
    if [ $lib = v1 ]; then export GTK_LIB_PATH=$PWD/ab/v1/libgtopk_b200.so; else unset GTK_LIB_PATH; fi
    GTK_PIPE_CHAIN=$chain python bench.py --steps 200 --warmup 20 --no-cpu 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib chain=$chain', d['value'], d['roofline']['launch_ms'], d['kernels_per_step'], d['stages_ms'])" >> gpurun_out/ab_chain.txt
  done
done
done
