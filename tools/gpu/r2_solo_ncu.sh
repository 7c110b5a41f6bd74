OUT=gpurun_out/solo_ncu
mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 5 -c 1 \
    -o $OUT/exchange_k270_solo python tools/exchange_latency.py --k 270 --P 2 --calls 8 > $OUT/ncu.log 2>&1
python tools/ncu_lines2.py $OUT/exchange_k270_solo.ncu-rep 40 > $OUT/lines.txt 2>&1
ncu -i $OUT/exchange_k270_solo.ncu-rep --page details --csv > $OUT/details.csv 2>&1
