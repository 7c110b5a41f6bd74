OUT=gpurun_out/api
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > $OUT/gpu_tests.txt
API_PROFILE=1 timeout 600 python tools/api_probe.py 25600000 25600 > $OUT/probe_headline.txt 2>&1
API_PROFILE=1 timeout 600 python tools/api_probe.py 270000 270 > $OUT/probe_r20.txt 2>&1
