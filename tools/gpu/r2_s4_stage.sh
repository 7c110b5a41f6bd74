# LL staging loads batched (one round trip per staging batch): loopback latency A/B
OUT=gpurun_out/s4_stage
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange_loopback.py -x -q > $OUT/pytest_loopback.txt 2>&1; echo "rc=$?" >> $OUT/pytest_loopback.txt
for cfg in "0 -1" "16 1" "8 1"; do
  set -- $cfg
  GTK_MERGE_GRID=$1 GTK_MERGE_CLUSTER=$2 timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 > $OUT/lat_g$1_c$2.jsonl 2>&1
done
timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 --deferred > $OUT/lat_deferred.jsonl 2>&1
timeout 300 python tools/exchange_latency.py --P 2 4 --k 2560 256000 > $OUT/lat_other_k.jsonl 2>&1
