# two GPUs: the multi-GPU suite with merge_solo on the real NVLink exchange,
# and BASELINE config 2 (ResNet-20, k = 270: the latency-bound merge path) / 1 / 3
OUT=gpurun_out/solo_multi
mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt
timeout 900 python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3 > $OUT/dist.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29991 \
    tools/sweep.py --configs 2,3,4 --no-cpu --out $OUT/sweep_n2.jsonl > $OUT/sweep_n2.log 2>&1
