#!/bin/bash
# Build an ablation copy of libexsum_b200.so with some translation units
# recompiled under extra -D flags:
#   tools/build_variant.sh OUT.so a.cu[,b.cu...] -DFOO=1 ...
# (load it with EXSUM_LIB=OUT.so; the default build is untouched)
set -e
out=$(realpath -m "$1"); srcs=$2; shift 2
cd "$(dirname "$0")/../paper_2106_00124_b200/csrc"
make -s -j8 >/dev/null
tmp=$(mktemp -d)
objs=$(ls build/*.o)
for src in ${srcs//,/ }; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
       -c "$src" -o "$tmp/${src%.cu}.o" 2>&1 | grep -v spill || true
  objs=$(echo "$objs" | grep -v "build/${src%.cu}.o")
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs "$tmp"/*.o
rm -rf "$tmp"
