nvidia-smi -L
python -m pytest tests/test_bench_protocol.py -x -q 2>&1 | tail -5 > gpurun_out/s1_proto_test.txt
python tools/sweep.py --protocol --out gpurun_out/r2_sweep_n1.jsonl > gpurun_out/r2_sweep_n1.log 2>&1
