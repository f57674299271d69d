#!/bin/bash
# Compiles the reference's own unit tests (proj/tests/test_*.cpp, unmodified,
# read in place under /root/reference) against this repository's drop-in C++
# API (include/ermc_b200.hpp via the ermc/*.hpp shims here) and links them to
# libermc_b200.so. Outputs go to tests/_refcompat/ (git-ignored; the binaries
# travel to the GPU box, where tests/test_gpu_refcompat.py runs them).
# TEST INFRASTRUCTURE: needs /root/reference (this container only).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF=${REF:-/root/reference/proj}
OUT=$ROOT/tests/_refcompat
mkdir -p "$OUT"
[ -d "$REF/tests" ] || { echo "no reference tree at $REF"; exit 0; }
g++ -std=c++20 -O1 -I"$HERE" -I"$ROOT/include" -c "$REF/tests/doctest_main.cpp" -o "$OUT/doctest_main.o"
for T in ${TESTS:-test_solver test_spectral test_geometry test_io test_sampling test_tracer}; do
  g++ -std=c++20 -O1 -I"$HERE" -I"$ROOT/include" -c "$REF/tests/$T.cpp" -o "$OUT/$T.o"
  g++ -o "$OUT/$T" "$OUT/$T.o" "$OUT/doctest_main.o" -L"$ROOT/paper_1810_00188_b200" -lermc_b200 \
      -Wl,-rpath,'$ORIGIN/../../paper_1810_00188_b200'
done
