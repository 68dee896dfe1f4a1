#!/usr/bin/env bash
# Builds the reference's own code into oracle/_ref/ (test infrastructure):
#   libref_rng.so    the reference's rng.cpp (the one TU that needs no Eigen) + ref_shim.cpp
#   libref_mcmp2.so  the reference's rng, gaussian, model, weights, sampler, greens, estimator,
#                    driver and oracle .cpp against oracle/eigen_subset (a minimal dense header written
#                    here: Eigen3 is absent from this image) + ref_mcmp2_shim.cpp; unmodified but
#                    for two sequenced reads in a copy of model.cpp (see below)
# Needs /root/reference (this container only); outputs go to oracle/_ref/ (git-ignored, but
# shipped to the GPU box with the snapshot). The reference's CMake build is not used.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${MCMP2_REFERENCE:-/root/reference}/proj/core"
if [ ! -f "$ref/src/rng.cpp" ]; then
  echo "build_ref: reference sources not present, skipping" >&2
  exit 0
fi
mkdir -p "$here/_ref"
g++ -std=c++20 -O2 -fPIC -shared -I"$ref/include" "$ref/src/rng.cpp" "$here/ref_shim.cpp" \
    -o "$here/_ref/libref_rng.so"
echo "built $here/_ref/libref_rng.so"
# model.cpp:295 and :310 read a point as Vec3(r.next_double(), r.next_double(), r.next_double()):
# the order in which C++ evaluates function arguments is unspecified, and g++ (the only compiler
# here) evaluates them right to left, reading every nucleus and basis centre as (z, y, x) -- for
# any centre off the origin the loaded set then fails its own orthonormality check. The recipe
# compiles a copy of model.cpp with the three reads sequenced left to right (the evident intent,
# and what a left-to-right compiler does); every other file is compiled as it lies.
mkdir -p "$here/_ref/src"
sed -e 's/Vec3(r\.next_double(), r\.next_double(), r\.next_double())/[\&] { const double x_ = r.next_double(), y_ = r.next_double(); return Vec3(x_, y_, r.next_double()); }()/' \
    -e 's/const Vec3 center(r\.next_double(), r\.next_double(), r\.next_double());/const Vec3 center = [\&] { const double x_ = r.next_double(), y_ = r.next_double(); return Vec3(x_, y_, r.next_double()); }();/' \
    "$ref/src/model.cpp" > "$here/_ref/src/model.cpp"
test "$(diff "$ref/src/model.cpp" "$here/_ref/src/model.cpp" | grep -c '^>')" = 2
srcs="$here/_ref/src/model.cpp"
for f in rng gaussian weights sampler greens estimator driver oracle; do srcs="$srcs $ref/src/$f.cpp"; done
g++ -std=c++20 -O2 -fPIC -shared -fvisibility=hidden -fvisibility-inlines-hidden -Wl,-Bsymbolic \
    -I"$here/eigen_subset" -I"$ref/include" $srcs "$here/ref_mcmp2_shim.cpp" -o "$here/_ref/libref_mcmp2.so" -lpthread
echo "built $here/_ref/libref_mcmp2.so"
# the reference's own unit tests (tests/test_*.cpp), built against oracle/doctest_subset
# (doctest is not vendored) and run by tests/test_reference_pins.py
tests="${MCMP2_REFERENCE:-/root/reference}/proj/tests"
if [ -f "$tests/test_rng.cpp" ]; then
  printf '#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include <doctest.h>\n' > "$here/_ref/src/test_main.cpp"
  tsrcs="$here/_ref/src/test_main.cpp"
  for f in rng model weights greens estimator sampler driver oracle; do tsrcs="$tsrcs $tests/test_$f.cpp"; done
  g++ -std=c++20 -O2 -I"$here/doctest_subset" -I"$here/eigen_subset" -I"$ref/include" -I"$tests" \
      $srcs $tsrcs -o "$here/_ref/ref_unit_tests" -lpthread
  echo "built $here/_ref/ref_unit_tests"
fi
