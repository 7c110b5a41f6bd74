# verify the current tree on 2 GPUs: full GPU suite, smoke(), bench N = 1 and N = 2
nvidia-smi -L
OUT=gpurun_out/s4_verify
mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29921 bench.py --gpus 2 --steps 200 --warmup 20 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
