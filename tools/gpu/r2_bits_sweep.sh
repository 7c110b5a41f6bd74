# one GPU: deferred select A/B at the bench's own preconditioning -- no
# bitmap (round-2 form), bitmap + release after the correction, bitmap +
# early release (finish grid 60 / 40)
OUT=gpurun_out/bits_sweep2
mkdir -p $OUT
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench_$name.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$name.json').read().strip().splitlines()[-1]); print('$name', d['value'], d['roofline']['frac'])" >> $OUT/summary.txt
}
run nobits GTK_DEFER_BITS=0
run bits_late GTK_DEFER_EARLY=0
run bits_early GTK_DEFER_EARLY=1
run bits_early_g40 GTK_DEFER_EARLY=1 GTK_FINISH_G=40
run nobits2 GTK_DEFER_BITS=0
