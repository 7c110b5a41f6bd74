# source-level stall profile of the exchange's merge: 16-CTA cluster vs 100-block grid, k = 25.6K, P = 2
OUT=gpurun_out/s4_ncu
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
GTK_MERGE_GRID=16 GTK_MERGE_CLUSTER=1 ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 5 -c 1 \
    -o $OUT/exchange_c16 python tools/exchange_latency.py --k 25600 --P 2 --calls 8 > $OUT/ncu_c16.log 2>&1
python tools/ncu_lines2.py $OUT/exchange_c16.ncu-rep 45 > $OUT/lines_c16.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 5 -c 1 \
    -o $OUT/exchange_g100 python tools/exchange_latency.py --k 25600 --P 2 --calls 8 > $OUT/ncu_g100.log 2>&1
python tools/ncu_lines2.py $OUT/exchange_g100.ncu-rep 45 > $OUT/lines_g100.txt 2>&1
