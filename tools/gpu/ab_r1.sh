# A/B on one B200: round-1 tree (ab/r1tree) vs the current tree, N=1 bench
nvidia-smi -L
for rep in 1 2 3; do
  (cd ab/r1tree && python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r1', d['value'], d['roofline']['launch_ms'], d.get('kernels_per_step'))") >> gpurun_out/ab_r1.txt
  for chain in 1 0; do
    GTK_PIPE_CHAIN=$chain python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cur chain=$chain', d['value'], d['roofline']['launch_ms'], d['kernels_per_step'])" >> gpurun_out/ab_r1.txt
  done
done
