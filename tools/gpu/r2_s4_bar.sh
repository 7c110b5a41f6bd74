# rotating-counter grid barrier: full GPU suite (incl. the 2-GPU tests), bench N = 1 / 2, loopback
# latency; then the previous {count, generation} barrier (GTK_GRID_BAR_GEN=1) for A/B on the same box
nvidia-smi -L
OUT=gpurun_out/s4_bar
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
ab() {
  tag=$1
  timeout 300 python tools/exchange_latency.py --P 2 4 8 --k 2560 25600 > $OUT/lat_$tag.jsonl 2>&1
  timeout 600 python bench.py --steps 200 --warmup 20 > $OUT/bench_n1_$tag.json 2> $OUT/bench_n1_$tag.err
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29913 bench.py --gpus 2 --steps 200 --warmup 20 > $OUT/bench_n2_$tag.json 2> $OUT/bench_n2_$tag.err
}
ab ctr
make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS=-DGTK_GRID_BAR_GEN=1 > $OUT/build_gen.log 2>&1
ab gen
make clean > /dev/null; make -j8 all > /dev/null 2>&1
ab ctr2
