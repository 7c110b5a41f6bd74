# cooperative vs plain (PDL) launches of the finish and the deferred exchange:
# does a cooperative launch start only after its predecessor completes?
nvidia-smi -L
OUT=gpurun_out/s4_coop
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python tools/defer_timeline.py > $OUT/timeline_n1_$tag.txt 2>&1
  env "$@" timeout 600 python bench.py --steps 200 --warmup 20 > $OUT/bench_n1_$tag.json 2> $OUT/bench_n1_$tag.err
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29911 tools/defer_timeline.py > $OUT/timeline_n2_$tag.txt 2>&1
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29913 bench.py --gpus 2 --steps 200 --warmup 20 > $OUT/bench_n2_$tag.json 2> $OUT/bench_n2_$tag.err
}
run base X=1
run xnc GTK_MERGE_COMPACT_COOP=0
run fnc GTK_FINISH_COOP=0
run both GTK_MERGE_COMPACT_COOP=0 GTK_FINISH_COOP=0
