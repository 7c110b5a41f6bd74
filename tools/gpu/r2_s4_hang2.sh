# after the soak-loop fix and the compact-grid default (32 + 24 per further round): repeated N = 4 / N = 2 bench runs
nvidia-smi -L
OUT=gpurun_out/s4_hang2
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
for i in 1 2 3 4 5 6 7 8; do
  n=$(( i % 2 == 0 ? 2 : 4 ))
  s=$(date +%s)
  GTK_HANG_DUMP=100 timeout 160 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29100 + i * 7)) bench.py --gpus $n --steps 200 --warmup 20 > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  echo "i=$i n=$n rc=$? $(( $(date +%s) - s ))s $(python -c "import json; d=json.loads(open('$OUT/bench_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])" 2>/dev/null)" >> $OUT/summary.txt
done
timeout 300 python -m pytest tests/test_gpu_dist.py -x -q > $OUT/dist.txt 2>&1; echo "rc=$?" >> $OUT/dist.txt
