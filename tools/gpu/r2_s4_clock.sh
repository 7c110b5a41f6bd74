# SM clock during the loopback exchange latency runs (clock64 / globaltimer of block 0)
OUT=gpurun_out/s4_clock
mkdir -p $OUT
make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS=-DGTK_MERGE_TRACE_FINE > $OUT/build.log 2>&1
export GTK_TRACE_FINE=1
timeout 300 python tools/exchange_latency.py --P 2 --k 270 25600 > $OUT/lat.jsonl 2>&1
GTK_MERGE_GRID=16 GTK_MERGE_CLUSTER=1 timeout 300 python tools/exchange_latency.py --P 2 --k 25600 > $OUT/lat_c16.jsonl 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/smi.txt
