# round 2, session 4: re-verify the restored tree on one B200 (suite, bench) and
# A/B the merge grid vs a thread-block cluster at k = 25.6K (loopback exchange)
OUT=gpurun_out/s4_first
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for cfg in "100 0" "16 1" "12 1" "8 1"; do
  set -- $cfg
  GTK_MERGE_GRID=$1 GTK_MERGE_CLUSTER=$2 timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 > $OUT/lat_g$1_c$2.jsonl 2>&1
done
