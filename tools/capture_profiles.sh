#!/bin/bash
# GPU-box recipe for the committed evidence under profiles/ (run via gpurun):
#   launch list of the bench command (steady state), full ncu sets of the
#   main pass (real L2 state), finish, merge and the sample kernel.
set -u
OUT=gpurun_out/prof_r1
mkdir -p $OUT
python bench.py --steps 200 --warmup 20 > $OUT/bench_n1.log 2>&1
# launch list: skip the preconditioning launches, keep ~50 steady steps
ncu --metrics gpu__time_duration.sum --clock-control none -s 6300 -c 220 --csv \
    --log-file $OUT/bench_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/ncu_launches.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:select_main_kernel -s 302 -c 1 \
    -o $OUT/select_main python tools/steady_main.py 300 > $OUT/ncu_main.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:select_finish_kernel -s 302 -c 1 \
    -o $OUT/select_finish python tools/steady_main.py 300 > $OUT/ncu_finish.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_sample_kernel -s 2 -c 1 \
    -o $OUT/select_sample python tools/prof_select.py 25600000 25600 3 > $OUT/ncu_sample.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 3 -c 1 \
    -o $OUT/merge python tools/prof_merge.py 25600 > $OUT/ncu_merge.log 2>&1
ls -la $OUT
