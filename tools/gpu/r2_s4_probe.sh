OUT=gpurun_out/s4_probe; mkdir -p $OUT; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $OUT/lat_probe tools/probe/lat_probe.cu && timeout 120 $OUT/lat_probe > $OUT/lat_probe.txt 2>&1
