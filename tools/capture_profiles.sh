#!/bin/bash
# GPU-box recipe for the committed evidence under profiles/ (run via gpurun,
# one GPU): the bench line, the launch list of the bench command (steady
# state), ncu --set full of the main pass (real L2 state), the finish, the
# sample kernel and the merge, main-pass timings at three sizes, finish
# phase traces.
set -u
OUT=gpurun_out/prof_r1
mkdir -p $OUT
python bench.py --steps 200 --warmup 20 > $OUT/bench_n1.json 2> $OUT/bench_n1.err
# launch list: skip the preconditioning launches (3 per step), keep ~50 steady steps
ncu --metrics gpu__time_duration.sum --clock-control none -s 4560 -c 150 --csv \
    --log-file $OUT/bench_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/ncu_launches.log 2>&1
python tools/launches.py $OUT/bench_launches.csv > $OUT/bench_launches_summary.txt
ncu --set full --cache-control none --clock-control none --import-source on -k regex:select_main_kernel -s 302 -c 1 \
    -o $OUT/select_main python tools/steady_main.py 300 > $OUT/ncu_main.log 2>&1
python tools/ncu_traffic.py $OUT/select_main.ncu-rep $OUT/select_main_ncu.json \
    "ncu --set full --cache-control none --clock-control none, steady-state residual (tools/steady_main.py 300, launch 303)"
ncu --set full --cache-control none --clock-control none --import-source on -k regex:select_finish_kernel -s 302 -c 1 \
    -o $OUT/select_finish python tools/steady_main.py 300 > $OUT/ncu_finish.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_sample_kernel -s 2 -c 1 \
    -o $OUT/select_sample python tools/prof_select.py 25600000 25600 3 > $OUT/ncu_sample.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 3 -c 1 \
    -o $OUT/merge python tools/prof_merge.py 25600 > $OUT/ncu_merge.log 2>&1
for r in select_main select_finish select_sample merge; do
  echo "== $r"; python tools/ncu_summary.py $OUT/$r.ncu-rep
done > $OUT/ncu_full_summary.txt 2>&1
python tools/ncu_lines2.py $OUT/select_main.ncu-rep 25 > $OUT/select_main_lines.txt 2>&1
python tools/ncu_lines2.py $OUT/select_finish.ncu-rep 25 > $OUT/select_finish_lines.txt 2>&1
for a in "25600000 25600" "14700000 14700" "66000000 66000" "66000000 660000"; do
  python tools/main_timing.py $a 1500
done > $OUT/main_timing.txt 2>&1
{ python tools/steady_trace.py 25600000 25600 1500; python tools/steady_trace.py 66000000 660000 400; } \
    > $OUT/finish_trace.txt 2>&1
python tools/merge_trace.py 25600 660000 > $OUT/merge_trace.txt 2>&1
ls -la $OUT
