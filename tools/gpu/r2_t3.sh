nvidia-smi -L
python -m pytest tests/test_gpu_exchange_loopback.py -x -q 2>&1 | tail -30 > gpurun_out/t3_loop.txt
python tools/exchange_latency.py --k 270 2560 25600 --P 2 4 > gpurun_out/t3_lat.jsonl 2>&1
GTK_MERGE_CLUSTER=0 python tools/exchange_latency.py --k 270 2560 25600 --P 2 > gpurun_out/t3_lat_grid.jsonl 2>&1
python -m pytest tests/test_gpu_kernels.py -x -q -k "chained" 2>&1 | tail -5 > gpurun_out/t3_chain.txt
python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/t3_bench.txt 2>&1
