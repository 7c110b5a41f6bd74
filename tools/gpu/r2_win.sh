OUT=gpurun_out/win
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "fallback or steady or deferred" 2>&1 | tail -4 > $OUT/tests_focus.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > $OUT/gpu_tests.txt
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench.json 2> $OUT/bench.err
