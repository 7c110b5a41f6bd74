# one GPU: merge / exchange parity with the one-CTA merge_solo path, then
# loopback latency (P = 2, 8; k = 270 .. 2048, one CTA up to 4096 union slots)
OUT=gpurun_out/solo
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_exchange_loopback.py tests/test_gpu_collectives.py -x -q 2>&1 | tail -15 > $OUT/tests.txt
for P in 2 8; do
  timeout 300 python tools/exchange_latency.py --P $P --k 270 1000 2048 > $OUT/lat_solo_p$P.jsonl 2>&1
done
timeout 300 python tools/exchange_latency.py --P 2 --k 270 1000 --deferred > $OUT/lat_solo_def.jsonl 2>&1
