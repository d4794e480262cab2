#!/bin/bash
# Build a variant of libanovafs.so with extra nvcc defines for A/B tuning runs:
#   tools/build_variant.sh NAME -DAFS_TC_U=1 ...   -> build_variants/libanovafs_NAME.so
# (select it with AFS_LIB=build_variants/libanovafs_NAME.so).  Reuses the objects of the
# main build (python -m paper_2111_10140_b200.build) for files without the defines' effect.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build_variants/$name
mkdir -p "$out"
for src in paper_2111_10140_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -I include -dc "$src" -o "$out/$(basename "${src%.cu}").o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC "$out"/*.o \
  -o "build_variants/libanovafs_$name.so" -lcudart_static -lpthread -ldl -lrt
echo "build_variants/libanovafs_$name.so"
