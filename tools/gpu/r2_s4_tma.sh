# main pass: bulk-copy (TMA) loads into shared memory (default) vs float4 register loads (GTK_MAIN_TMA=0)
nvidia-smi -L
OUT=gpurun_out/s4_tma
mkdir -p $OUT
ab() {
  tag=$1
  for i in 1 2; do timeout 600 python bench.py --steps 200 --warmup 20 > $OUT/bench_n1_${tag}_$i.json 2> $OUT/bench_n1_${tag}_$i.err; done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29941 bench.py --gpus 2 --steps 200 --warmup 20 > $OUT/bench_n2_$tag.json 2> $OUT/bench_n2_$tag.err
  timeout 300 python tools/defer_timeline.py > $OUT/timeline_n1_$tag.txt 2>&1
}
make -j8 all > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_recipes.py tests/test_gpu_collectives.py -x -q > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
ab tma
make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS=-DGTK_MAIN_TMA=0 > $OUT/build_reg.log 2>&1
ab reg
make clean > /dev/null; make -j8 all > /dev/null 2>&1
ab tma2
