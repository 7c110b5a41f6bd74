OUT=gpurun_out/tau2
mkdir -p $OUT
GTK_E2E_DEBUG=1 timeout 600 python bench.py --no-cpu --steps 40 --warmup 5 > $OUT/bench_dbg.json 2> $OUT/bench_dbg.err
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > $OUT/gpu_tests.txt
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench.json 2> $OUT/bench.err
