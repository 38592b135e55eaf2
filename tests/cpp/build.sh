#!/bin/sh
# Builds tests/cpp/dropin_parity (TEST INFRASTRUCTURE): the reference's core
# objects (oracle/_ref, built by `make -C oracle ref`) + this repo's shim over
# libpstereo_gpu.so. Needs /root/reference (headers); output in build/.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${REF:-/root/reference/proj}
[ -d "$REF/include" ] || { echo "no reference headers at $REF"; exit 0; }
make -s -C "$ROOT/oracle" ref
mkdir -p "$ROOT/build"
O="$ROOT/oracle/_ref"
g++ -std=gnu++20 -O2 -I"$REF/include" -I"$ROOT/include" "$ROOT/tests/cpp/dropin_parity.cpp" \
  "$O/image.o" "$O/pyramid.o" "$O/patch.o" "$O/lk_solver.o" "$O/window_posterior.o" \
  "$O/spatial_mask.o" "$O/coarse_to_fine.o" "$O/depth_variance.o" "$O/pipeline.o" \
  -L"$ROOT/paper_2205_03133_b200" -lpstereo_gpu -Wl,-rpath,'$ORIGIN/../paper_2205_03133_b200' \
  -lpthread -o "$ROOT/build/dropin_parity"
g++ -std=gnu++20 -O2 -I"$REF/include" -I"$ROOT/include" "$ROOT/tests/cpp/dropin_bench.cpp" \
  "$O/image.o" "$O/pyramid.o" "$O/patch.o" "$O/lk_solver.o" "$O/window_posterior.o" \
  "$O/spatial_mask.o" "$O/coarse_to_fine.o" "$O/depth_variance.o" "$O/pipeline.o" \
  "$O/metrics.o" "$O/synth.o" "$O/bench.o" "$O/ref_glue.o" \
  -L"$ROOT/paper_2205_03133_b200" -lpstereo_gpu -Wl,-rpath,'$ORIGIN/../paper_2205_03133_b200' \
  -lpthread -o "$ROOT/build/dropin_bench"
echo "built $ROOT/build/dropin_parity $ROOT/build/dropin_bench"
