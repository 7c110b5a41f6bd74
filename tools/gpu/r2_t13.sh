nvidia-smi -L
python -m pytest tests -q -m gpu -x 2>&1 | tail -8 > gpurun_out/t13_all.txt
python tools/defer_timeline.py > gpurun_out/t13_tl.txt 2>&1
python bench.py --steps 200 --warmup 20 > gpurun_out/t13_bench.txt 2>&1
GTK_PIPE_MODE=chain python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | tail -1 > gpurun_out/t13_bench_chain.txt
