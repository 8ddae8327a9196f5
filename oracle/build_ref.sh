#!/usr/bin/env bash
# Build the reference's OWN sources (unmodified, compiled where they lie under
# /root/reference) against the Eigen-subset shim into oracle/_ref/.
# ORACLE TEST INFRASTRUCTURE ONLY. Outputs only into oracle/_ref/ (gitignored,
# not gpurun-ignored: the prebuilt .so travels to the GPU box).
# Flags follow the reference's Release build (proj/CMakeLists.txt, src/CMakeLists.txt):
# C++20, -O3 -DNDEBUG, kernels_avx2.cpp selects AVX2/FMA by function attributes.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF=/root/reference/proj
OUT="$HERE/_ref"
[ -d "$REF/src" ] || { echo "reference not present; skipping"; exit 0; }
mkdir -p "$OUT"
SRCS="tensorops fdsolver eigensolve krylov kernels kernels_avx2 assembly bspline problems experiments"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -w -I$HERE/eigen_shim -I$REF/include"
objs=()
for s in $SRCS; do
  o="$OUT/$s.o"
  if [ ! -f "$o" ] || [ "$REF/src/$s.cpp" -nt "$o" ] || [ "$HERE/eigen_shim/Eigen/Core" -nt "$o" ] || [ "$HERE/eigen_shim/Eigen/Dense" -nt "$o" ]; then
    $CXX $FLAGS -c "$REF/src/$s.cpp" -o "$o" &
  fi
  objs+=("$o")
done
wait
$CXX $FLAGS -c "$HERE/ref_driver.cpp" -o "$OUT/ref_driver.o"
$CXX -shared -o "$OUT/libkronschro_ref.so" "${objs[@]}" "$OUT/ref_driver.o"
echo "built $OUT/libkronschro_ref.so"
# the reference-side binding as a runnable drop-in demo,
# linked against the reference objects and libks.so (rpath = repo-relative)
KS="$HERE/../paper_2311_18461_b200"
if [ -f "$KS/libks.so" ]; then
  $CXX $FLAGS -I"$HERE/../include" "$HERE/integration_demo.cpp" "${objs[@]}" -o "$OUT/integration_demo" \
      -L"$KS" -lks -Wl,-rpath,'$ORIGIN/../../paper_2311_18461_b200'
  echo "built $OUT/integration_demo"
fi
