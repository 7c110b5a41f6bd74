# deferred exchange compact grid: the new default (32 + 16 per further merge round) vs neighbours at N = 4
nvidia-smi -L
OUT=gpurun_out/s4_cg2
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
run() {  # n g(0 = default)
  if [ "$2" = 0 ]; then E=X=1; else E=GTK_MERGE_COMPACT_G=$2; fi
  timeout 200 env $E python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29300 + $1 * 100 + $2)) bench.py --gpus $1 --steps 200 --warmup 20 > $OUT/bench_n$1_g$2.json 2> $OUT/bench_n$1_g$2.err
  echo "n=$1 g=$2 $(python -c "import json; d=json.loads(open('$OUT/bench_n$1_g$2.json').read().strip().splitlines()[-1]); print(d['value'])" 2>/dev/null)" >> $OUT/summary.txt
}
for g in 0 40 56 0; do run 4 $g; done
run 2 0
timeout 300 python -m pytest tests/test_gpu_dist.py -x -q > $OUT/dist.txt 2>&1; echo "rc=$?" >> $OUT/dist.txt
