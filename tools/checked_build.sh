#!/bin/bash
# The bounds-checked library (GTK_CHECKED: every shared / global index the
# kernels compute asserted in range) -> ab/checked/libgtopk_b200.so; run the
# GPU suite against it with GTK_LIB_PATH=$PWD/ab/checked/libgtopk_b200.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/checked ab/checked
for f in paper_1901_04359_b200/csrc/*.cu; do
  b=$(basename "$f" .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -DGTK_CHECKED -c "$f" -o "build/checked/$b.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/checked/libgtopk_b200.so build/checked/*.o
echo "built ab/checked/libgtopk_b200.so"
