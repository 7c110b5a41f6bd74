# one GPU, same box: the correction's inputs preloaded (working tree) vs HEAD (ab/pre)
OUT=$PWD/gpurun_out/fixpre_ab
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_recipes.py -x -q 2>&1 | tail -3 > $OUT/tests.txt
run() {  # name, dir
  (cd $2 && timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench_$1.json 2>/dev/null)
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$1.json').read().strip().splitlines()[-1]); print('$1', d['value'], d['roofline']['frac'])" >> $OUT/summary.txt
}
run pre ab/pre
run new .
run pre2 ab/pre
run new2 .
timeout 300 python tools/defer_timeline.py > $OUT/timeline.txt 2>&1
