#!/bin/sh
# Development tool: build an A/B variant of the product library that differs
# only in bdis_patches.cu compile definitions (after a normal build, which
# provides the other objects). Usage: variant.sh NAME -DKEY=VAL ...
# -> build/var/NAME/libpstereo_gpu.so (select with PSTEREO_GPU_LIB).
# SRC=path compiles another copy of the file (e.g. `git show HEAD:...` output).
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
NAME=$1; shift
OUT=$ROOT/build/var/$NAME
mkdir -p "$OUT"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -I "$ROOT/paper_2205_03133_b200/csrc" \
  -Xcompiler -fPIC -Xptxas -v "$@" -c "${SRC:-$ROOT/paper_2205_03133_b200/csrc/bdis_patches.cu}" \
  -o "$OUT/bdis_patches.cu.o" 2> "$OUT/ptxas.log"
OBJS=""
for o in bdis_kernels.cu bdis_metrics.cu bdis_capi.cu bdis_synth.cu bdis_render.cu synth.c host_io.cpp bdis_multi.cpp host_expand.cpp; do
  OBJS="$OBJS $ROOT/build/obj/$o.o"
done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libpstereo_gpu.so" \
  "$OUT/bdis_patches.cu.o" $OBJS -lpthread -lm -lz
grep -A3 "Compiling entry function '_ZN4bdis9k_patchesILi8ELb1ELb0" "$OUT/ptxas.log" | tail -2
