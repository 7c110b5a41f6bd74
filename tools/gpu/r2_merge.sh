# merge-latency survey on one B200 (loopback exchange) + main-pass A/B
nvidia-smi -L
python tools/exchange_latency.py --k 270 2560 25600 --P 2 4 > gpurun_out/lat_auto.jsonl 2>&1
GTK_MERGE_CLUSTER=0 python tools/exchange_latency.py --k 270 2560 25600 --P 2 4 > gpurun_out/lat_grid.jsonl 2>&1
for g in 1 2 4 8 16; do
  GTK_MERGE_CLUSTER=1 GTK_MERGE_GRID=$g python tools/exchange_latency.py --k 270 2560 25600 --P 2 > gpurun_out/lat_c$g.jsonl 2>&1
done
for rep in 1 2; do
  python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cur', d['value'], d['roofline']['launch_ms'], d['kernels_per_step'])" >> gpurun_out/ab_main.txt
  GTK_LIB_PATH=$PWD/ab/p0/libgtopk_b200.so python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p0', d['value'], d['roofline']['launch_ms'], d['kernels_per_step'])" >> gpurun_out/ab_main.txt
  (cd ab/r1tree && python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r1', d['value'], d['roofline']['launch_ms'], d.get('kernels_per_step'))") >> gpurun_out/ab_main.txt
done
