# instruction fetch: loopback exchange latency with the kernel's code L2-resident vs evicted (512 MB streamed
# through L2 before each call)
OUT=gpurun_out/s4_thrash
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
for t in 0 512; do
  timeout 300 python tools/exchange_latency.py --P 2 4 --k 270 25600 --thrash-mb $t > $OUT/lat_t$t.jsonl 2>&1
  timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 --deferred --thrash-mb $t > $OUT/lat_def_t$t.jsonl 2>&1
done
