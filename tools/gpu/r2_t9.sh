nvidia-smi -L
V=$PWD/ab/fmb3/libgtopk_b200.so
GTK_LIB_PATH=$V GTK_DEFER_EARLY=1 python tools/defer_timeline.py > gpurun_out/t9_tl_fmb3.txt 2>&1
for rep in 1 2; do
  for cfg in "early=1 mb=2" "early=1 mb=3" "early=0 mb=3" "chain mb=3" "chain mb=2"; do
    env=""
    case "$cfg" in *"mb=3"*) env="GTK_LIB_PATH=$V";; esac
    case "$cfg" in early=1*) env="$env GTK_DEFER_EARLY=1";; early=0*) env="$env GTK_DEFER_EARLY=0";; chain*) env="$env GTK_PIPE_MODE=chain";; esac
    eval "$env python bench.py --steps 200 --warmup 20 --no-cpu" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['run']['dense_fallback_in_timed_steps'])" >> gpurun_out/t9_ab.txt
  done
done
