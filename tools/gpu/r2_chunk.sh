OUT=gpurun_out/chunk
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "pinned_host or public_step or dense_fallback" 2>&1 | tail -4 > $OUT/tests.txt
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python tools/probe/e2e_probe.py > $OUT/e2e_probe.txt 2>&1
