nvidia-smi -L
python -m pytest tests/test_gpu_exchange_loopback.py -x -q 2>&1 | tail -15 > gpurun_out/t14_loop.txt
python tools/exchange_latency.py --k 270 2560 25600 --P 2 4 8 > gpurun_out/t14_lat.jsonl 2>&1
python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/t14_all.txt
