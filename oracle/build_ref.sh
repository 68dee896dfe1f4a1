#!/usr/bin/env bash
# Builds oracle/_ref/libref_rng.so from the reference's own rng.cpp (the only reference TU that
# compiles without Eigen3; SURVEY.md finding 1) plus oracle/ref_shim.cpp. Test infrastructure:
# the library pins the oracle's Philox restatement. Needs /root/reference (this container only);
# outputs go to oracle/_ref/ (git-ignored, but shipped to the GPU box with the snapshot).
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
