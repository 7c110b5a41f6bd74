# one GPU, same box: select-workspace layout sensitivity of the N = 1 step
# (HEAD; + a 3.2 MB region in the middle of the workspace; + 3.2 MB at its end)
OUT=$PWD/gpurun_out/layout_ab
mkdir -p $OUT
run() {  # name, dir
  (cd $2 && timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 > $OUT/bench_$1.json 2>/dev/null)
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$1.json').read().strip().splitlines()[-1]); print('$1', d['value'], d['roofline']['frac'])" >> $OUT/summary.txt
}
run head .
run mid ab/lay_mid
run end ab/lay_end
run head2 .
run mid2 ab/lay_mid
