#!/bin/bash
# make + verify the library is newer than every source (guards against stale pushes)
set -e
cd "$(dirname "$0")/.."
make -j8 all > build/make.log 2>&1 || { cat build/make.log; exit 1; }
so=paper_1901_04359_b200/libgtopk_b200.so
for f in paper_1901_04359_b200/csrc/* include/*.h; do
  if [ "$f" -nt "$so" ]; then echo "STALE: $f newer than $so"; exit 1; fi
done
grep -h "registers\|spill" build/*.ptxas.txt | grep -v " 0 bytes spill stores" | grep spill || true
echo "build ok: $(stat -c %y $so)"
