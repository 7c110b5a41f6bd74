# development check on one B200 (gpurun): new tests first, then the suite, then the bench
set -x
TAG=${1:-t}
nvidia-smi -L
python -m pytest tests/test_gpu_kernels.py -k "chained" -x -q 2>&1 | tail -30 > gpurun_out/r2_${TAG}_chain.txt
python -m pytest tests/test_gpu_recipes.py -x -q 2>&1 | tail -30 > gpurun_out/r2_${TAG}_recipes.txt
python bench.py --steps 200 --warmup 20 > gpurun_out/r2_${TAG}_bench.txt 2>&1
python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r2_${TAG}_all.txt
