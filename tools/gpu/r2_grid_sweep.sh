# one GPU: loopback exchange latency at k = 25.6K vs merge grid size (merge-path union)
OUT=gpurun_out/grid_sweep
mkdir -p $OUT
for g in 32 50 64 100 128; do
  GTK_MERGE_GRID=$g timeout 300 python tools/exchange_latency.py --P 2 4 --k 25600 > $OUT/lat_g$g.jsonl 2>&1
done
