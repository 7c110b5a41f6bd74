#!/bin/bash
# GPU-box recipe for the round-2 evidence under profiles/ (one GPU, via gpurun):
# the bench line, the bench command's launch list (steady state), ncu --set full
# of the deferred main pass / finish in their steady state, of the exchange kernel
# (loopback, k = 25.6K and 270) and of the standalone merge, plus timelines.
set -u
OUT=${OUT:-gpurun_out/prof_r2}
mkdir -p $OUT
python bench.py --steps 200 --warmup 20 > $OUT/bench_n1.json 2> $OUT/bench_n1.err
# launch list: 300 preconditioning steps (2 launches each) + capture, then the timed steps
ncu --metrics gpu__time_duration.sum --clock-control none -s 640 -c 120 --csv \
    --log-file $OUT/bench_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --precondition 300 \
    > $OUT/ncu_launches.log 2>&1
python tools/launches.py $OUT/bench_launches.csv > $OUT/bench_launches_summary.txt
ncu --set full --cache-control none --clock-control none --import-source on -k regex:select_main_kernel -s 302 -c 1 \
    -o $OUT/select_main python tools/steady_main.py 300 > $OUT/ncu_main.log 2>&1
python tools/ncu_traffic.py $OUT/select_main.ncu-rep $OUT/select_main_ncu.json \
    "ncu --set full --cache-control none --clock-control none, deferred pipeline steady state (tools/steady_main.py 300, main launch 303)"
ncu --set full --cache-control none --clock-control none --import-source on -k regex:select_finish_kernel -s 302 -c 1 \
    -o $OUT/select_finish python tools/steady_main.py 300 > $OUT/ncu_finish.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 5 -c 1 \
    -o $OUT/exchange_k25600 python tools/exchange_latency.py --k 25600 --P 2 --calls 8 > $OUT/ncu_exchange.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 5 -c 1 \
    -o $OUT/exchange_k25600_deferred python tools/exchange_latency.py --k 25600 --P 2 --calls 8 --deferred \
    > $OUT/ncu_exchange_deferred.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 5 -c 1 \
    -o $OUT/exchange_k270 python tools/exchange_latency.py --k 270 --P 2 --calls 8 > $OUT/ncu_exchange270.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 3 -c 1 \
    -o $OUT/merge python tools/prof_merge.py 25600 > $OUT/ncu_merge.log 2>&1
for r in select_main select_finish exchange_k25600 exchange_k25600_deferred exchange_k270 merge; do
  echo "== $r"; python tools/ncu_summary.py $OUT/$r.ncu-rep
done > $OUT/ncu_full_summary.txt 2>&1
python tools/ncu_lines2.py $OUT/select_finish.ncu-rep 25 > $OUT/select_finish_lines.txt 2>&1
python tools/ncu_lines2.py $OUT/exchange_k25600.ncu-rep 25 > $OUT/exchange_lines.txt 2>&1
for mode in defer chain plain; do GTK_PIPE_MODE=$mode python tools/defer_timeline.py; done > $OUT/select_timelines.txt 2>&1
python tools/exchange_latency.py --k 270 2560 25600 --P 2 4 8 > $OUT/exchange_latency.jsonl 2>&1
python tools/exchange_latency.py --k 270 2560 25600 --P 2 4 8 --deferred > $OUT/exchange_latency_deferred.jsonl 2>&1
for a in "25600000 25600" "14700000 14700" "66000000 66000" "66000000 660000"; do
  python tools/main_timing.py $a 1500
done > $OUT/main_timing.txt 2>&1
ls -la $OUT
