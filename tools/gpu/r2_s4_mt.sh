# merge / exchange blocks of 256 threads (<= 128 registers: a main-pass block fits beside one) vs 512
nvidia-smi -L
OUT=gpurun_out/s4_mt
mkdir -p $OUT
run() {  # tag n
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
    --master-port $((29600 + $2 + ${#1})) bench.py --gpus $2 --steps 200 --warmup 20 > $OUT/bench_$1_n$2.json 2> $OUT/bench_$1_n$2.err
  echo "$1 n=$2 rc=$? $(python -c "import json,sys; d=json.loads(open('$OUT/bench_$1_n$2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])" 2>/dev/null)" >> $OUT/summary.txt
}
make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS=-DGTK_MERGE_THREADS=256 > $OUT/build256.log 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_collectives.py -x -q > $OUT/pytest256.txt 2>&1; echo "rc=$?" >> $OUT/pytest256.txt
timeout 300 python tools/exchange_latency.py --P 2 4 --k 270 2560 25600 > $OUT/lat256.jsonl 2>&1
timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 --deferred > $OUT/lat256_def.jsonl 2>&1
run t256 2; run t256 4
make clean > /dev/null; make -j8 all > $OUT/build512.log 2>&1
timeout 300 python tools/exchange_latency.py --P 2 4 --k 270 2560 25600 > $OUT/lat512.jsonl 2>&1
timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 --deferred > $OUT/lat512_def.jsonl 2>&1
run t512 2; run t512 4
make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS=-DGTK_MERGE_THREADS=256 > /dev/null 2>&1
run u256 2; run u256 4
