# diagnostic build (GTK_MERGE_TRACE_FINE): union-phase stamps of block 0
OUT=gpurun_out/s4_fine
mkdir -p $OUT
make clean > /dev/null; make -j8 all GTK_EXTRA_FLAGS=-DGTK_MERGE_TRACE_FINE > $OUT/build.log 2>&1
export GTK_TRACE_FINE=1
for cfg in "0 -1" "16 1" "32 0"; do
  set -- $cfg
  GTK_MERGE_GRID=$1 GTK_MERGE_CLUSTER=$2 timeout 300 python tools/exchange_latency.py --P 2 --k 25600 > $OUT/lat_g$1_c$2.jsonl 2>&1
done
timeout 300 python tools/exchange_latency.py --P 2 --k 25600 --deferred > $OUT/lat_deferred.jsonl 2>&1
