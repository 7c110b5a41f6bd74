# NVLink bytes of the exchange kernel on rank 0 of a 2-GPU gTopKAllReduce:
# rank 0 under ncu (single-pass metric set: nvltx/nvlrx bytes + duration), rank 1 plain
nvidia-smi -L
export WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=29811
RANK=1 LOCAL_RANK=1 timeout 300 python tools/nvl_exchange.py > gpurun_out/nvl_rank1.txt 2>&1 &
RANK=0 LOCAL_RANK=0 timeout 300 ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum \
  --clock-control none -c 60 --csv --log-file gpurun_out/nvl_ncu.csv \
  python tools/nvl_exchange.py > gpurun_out/nvl_rank0.txt 2>&1
wait
