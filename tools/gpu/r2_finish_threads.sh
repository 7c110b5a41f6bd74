# one GPU, same box: finish block size (512 threads = HEAD; 256 x 64 regs and
# 384 x 56 regs fit beside two main-pass blocks, so they land earlier in the drain)
OUT=$PWD/gpurun_out/finish_threads
mkdir -p $OUT
run() {  # name, dir, env...
  name=$1; dir=$2; shift 2
  (cd $dir && env "$@" timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench_$name.json 2>/dev/null)
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$name.json').read().strip().splitlines()[-1]); print('$name', d['value'], d['roofline']['frac'])" >> $OUT/summary.txt
}
run head . A=1
run t256 ab/t256 A=1
run t384 ab/t384 A=1
run t256_g40 ab/t256 GTK_FINISH_G=40
run t384_g40 ab/t384 GTK_FINISH_G=40
run head2 . A=1
(cd ab/t256 && timeout 300 python tools/defer_timeline.py > $OUT/timeline_t256.txt 2>&1)
