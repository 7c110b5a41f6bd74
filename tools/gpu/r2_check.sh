set -x
nvidia-smi -L
python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_recipes.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/r2_t1_new.txt
python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r2_t1_all.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_t1_bench.txt 2>&1
