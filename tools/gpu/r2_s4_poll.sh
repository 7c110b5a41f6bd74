# deferred finish: poll the main pass's done counter (default) vs griddepcontrol.wait (GTK_FINISH_POLL=0)
nvidia-smi -L
OUT=gpurun_out/s4_poll
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
ab() {
  tag=$1; shift
  for i in 1 2; do env "$@" timeout 600 python bench.py --steps 200 --warmup 20 > $OUT/bench_n1_${tag}_$i.json 2> $OUT/bench_n1_${tag}_$i.err; done
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29951 bench.py --gpus 2 --steps 200 --warmup 20 > $OUT/bench_n2_$tag.json 2> $OUT/bench_n2_$tag.err
  env "$@" timeout 300 python tools/defer_timeline.py > $OUT/timeline_n1_$tag.txt 2>&1
}
ab poll X=1
ab wait GTK_FINISH_POLL=0
ab poll2 X=1
