# merge_device with one engine call site (exchange_kernel 12.3K -> 8.2K SASS instructions): tests, loopback, bench N = 2 / 4
nvidia-smi -L
OUT=gpurun_out/s4_compact
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_collectives.py tests/test_gpu_kernels.py -x -q > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
timeout 300 python tools/exchange_latency.py --P 2 4 8 --k 270 2560 25600 > $OUT/lat.jsonl 2>&1
timeout 300 python tools/exchange_latency.py --P 2 4 8 --k 2560 25600 --deferred > $OUT/lat_def.jsonl 2>&1
timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 --thrash-mb 512 > $OUT/lat_t512.jsonl 2>&1
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n --steps 200 --warmup 20 > $OUT/bench_n$n.json 2> $OUT/bench_n$n.err
done
timeout 300 python -m pytest tests/test_gpu_dist.py -x -q > $OUT/dist.txt 2>&1; echo "rc=$?" >> $OUT/dist.txt
