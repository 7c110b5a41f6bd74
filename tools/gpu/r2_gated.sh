# one GPU: the gated deferred finish -- GPU suite, same-box A/B bench lines
# (GTK_DEFER_GATED=0 = the finish waits for the whole main pass), timelines
OUT=$PWD/gpurun_out/gated
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > $OUT/gpu_tests.txt
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench_$name.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$name.json').read().strip().splitlines()[-1]); print('$name', d['value'], d['roofline']['frac'])" >> $OUT/summary.txt
}
run gated A=1
run ungated GTK_DEFER_GATED=0
run gated2 A=1
timeout 300 python tools/defer_timeline.py > $OUT/timeline.txt 2>&1
