# merge round-0 histogram spread over more L2 lines (GTK_HIST_SPREAD words per bin): loopback latency per build
OUT=gpurun_out/s4_spread
mkdir -p $OUT
for sp in 1 4 16 32; do
  make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS="-DGTK_HIST_SPREAD=$sp -DGTK_MERGE_TRACE_FINE" > $OUT/build_$sp.log 2>&1
  GTK_TRACE_FINE=1 timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 > $OUT/lat_sp$sp.jsonl 2>&1
  GTK_TRACE_FINE=1 timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 --deferred > $OUT/lat_def_sp$sp.jsonl 2>&1
done
make clean > /dev/null; make -j8 all > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py tests/test_gpu_collectives.py -x -q > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
