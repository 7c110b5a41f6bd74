# deferred exchange: compact grid size sweep after the barrier change (GTK_MERGE_COMPACT_G)
nvidia-smi -L
OUT=gpurun_out/s4_cg
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
run() {  # n g
  timeout 200 env GTK_MERGE_COMPACT_G=$2 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29400 + $1 * 100 + $2)) bench.py --gpus $1 --steps 200 --warmup 20 > $OUT/bench_n$1_g$2.json 2> $OUT/bench_n$1_g$2.err
  echo "n=$1 g=$2 $(python -c "import json; d=json.loads(open('$OUT/bench_n$1_g$2.json').read().strip().splitlines()[-1]); print(d['value'])" 2>/dev/null)" >> $OUT/summary.txt
}
for g in 16 24 32 40 32; do run 2 $g; done
for g in 32 48 64 80 64; do run 4 $g; done
