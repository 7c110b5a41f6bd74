# one GPU, same box: HEAD before the winner bitmap (ab/pre) vs the working
# tree (no bitmap / bitmap + early release), bench lines without the CPU leg
OUT=$PWD/gpurun_out/bits_ab
mkdir -p $OUT
run() {  # name, dir, env...
  name=$1; dir=$2; shift 2
  (cd $dir && env "$@" timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench_$name.json 2>/dev/null)
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$name.json').read().strip().splitlines()[-1]); print('$name', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" >> $OUT/summary.txt
}
run pre ab/pre A=1
run new_nobits . GTK_DEFER_BITS=0
run new_bits . A=1
run pre2 ab/pre A=1
run new_bits2 . A=1
