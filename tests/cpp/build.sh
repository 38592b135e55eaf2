#!/bin/sh
# TEST INFRASTRUCTURE: builds the drop-in caller test (tests/cpp/caller_main.cpp)
# twice -- needs /root/reference (sources and headers) at build time; the
# binaries land in build/ and travel to the GPU box with the snapshot.
#
#   build/caller_ref  the unmodified reference: all of proj/src + the caller
#   build/caller_gpu  the reference's caller-side sources (bench, io, metrics,
#                     runner, synth -- unchanged) + the caller, compiled with
#                     this repo's include/ ahead of the reference's include/
#                     (the drop-in headers include/pstereo/*.hpp), linked
#                     against libpstereo_gpu.so instead of the matcher sources
#
# libpng and CLI11 are absent here: tests/cpp/stubs/ stands in for both
# (PGM/PPM input only; no command-line parsing).
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${REF:-/root/reference/proj}
[ -d "$REF/src" ] || { echo "no reference sources at $REF"; exit 0; }
CXX=${CXX:-g++}
FLAGS="-std=gnu++20 -O3 -DNDEBUG"
STUBS="$ROOT/tests/cpp/stubs"
B="$ROOT/build/dropin"
mkdir -p "$B/ref" "$B/gpu"
CALLERS="bench io metrics runner synth"
MATCHER="image pyramid patch lk_solver window_posterior spatial_mask coarse_to_fine depth_variance pipeline"

# the reference, whole
for s in $CALLERS $MATCHER; do
  o="$B/ref/$s.o"
  if [ ! -f "$o" ] || [ "$REF/src/$s.cpp" -nt "$o" ]; then
    $CXX $FLAGS -I"$STUBS" -I"$REF/include" -c "$REF/src/$s.cpp" -o "$o"
  fi
done
$CXX $FLAGS -I"$STUBS" -I"$REF/include" "$ROOT/tests/cpp/caller_main.cpp" \
  $(for s in $CALLERS $MATCHER; do echo "$B/ref/$s.o"; done) -lpthread -o "$ROOT/build/caller_ref"

# the drop-in: the same callers, this repo's headers first, no matcher sources
for s in $CALLERS; do
  $CXX $FLAGS -I"$STUBS" -I"$ROOT/include" -I"$REF/include" -c "$REF/src/$s.cpp" -o "$B/gpu/$s.o"
done
$CXX $FLAGS -I"$STUBS" -I"$ROOT/include" -I"$REF/include" "$ROOT/tests/cpp/caller_main.cpp" \
  $(for s in $CALLERS; do echo "$B/gpu/$s.o"; done) \
  -L"$ROOT/paper_2205_03133_b200" -lpstereo_gpu -Wl,-rpath,'$ORIGIN/../paper_2205_03133_b200' \
  -lpthread -o "$ROOT/build/caller_gpu"
echo "built $ROOT/build/caller_ref $ROOT/build/caller_gpu"
