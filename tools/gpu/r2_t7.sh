nvidia-smi -L
python tools/defer_debug.py 25600000 25600 12 > gpurun_out/defer_dbg.txt 2>&1
for mode in defer chain plain; do GTK_PIPE_MODE=$mode python tools/defer_timeline.py > gpurun_out/t7_tl_$mode.txt 2>&1; done
python -m pytest tests/test_gpu_kernels.py -x -q -k "deferred" 2>&1 | tail -5 > gpurun_out/t7_kern.txt
