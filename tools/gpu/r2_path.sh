# one GPU: merge-path union slots (solo and grid merges) -- GPU suite (normal
# and bounds-checked library), loopback exchange latency
OUT=gpurun_out/path
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > $OUT/gpu_tests.txt
GTK_LIB_PATH=$PWD/ab/checked/libgtopk_b200.so timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_exchange_loopback.py tests/test_gpu_collectives.py -x -q 2>&1 | tail -4 > $OUT/checked_tests.txt
timeout 600 python tools/exchange_latency.py --P 2 8 --k 270 1000 2048 25600 > $OUT/lat.jsonl 2>&1
timeout 600 python tools/exchange_latency.py --P 2 4 --k 25600 --deferred > $OUT/lat_def.jsonl 2>&1
