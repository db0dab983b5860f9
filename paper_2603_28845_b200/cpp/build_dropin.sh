#!/usr/bin/env bash
# Builds the C++ drop-in (paper_2603_28845_b200/cpp/ocw_dropin.cpp: the
# reference's ocw:: quantizer interface over libocwg.so) and links the
# reference's OWN unit tests against it, unmodified, from the read-only tree:
#   lib/libocw_dropin.so        ocw_dropin.cpp + proj/src/matrix.cpp (the Matrix type)
#   lib/dropin_test_core        proj/tests/test_core.cpp      -> GPU implementation
#   lib/dropin_test_layerwise   proj/tests/test_layerwise.cpp -> GPU implementation
#   lib/dropin_test_jointq      proj/tests/test_jointq.cpp    -> GPU implementation (f4)
# Outputs are build products (git-ignored) that travel to the GPU box.
set -euo pipefail
REF=${OCW_REFERENCE:-/root/reference/proj}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
PKG="$(dirname "$HERE")"
ROOT="$(dirname "$PKG")"
if [ ! -d "$REF/src" ]; then
  echo "build_dropin: $REF not present; skipping (prebuilt lib/ binaries are used if shipped)" >&2
  exit 0
fi
CXX=${CXX:-g++}
INC="-I$REF/include -I$PKG/compat -I$ROOT/oracle/shim -I$ROOT/include"
FLAGS="-std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter $INC"
LIB="$PKG/lib"
$CXX $FLAGS -shared -o "$LIB/libocw_dropin.so" "$HERE/ocw_dropin.cpp" "$REF/src/matrix.cpp" \
  -L"$LIB" -locwg -Wl,-rpath,'$ORIGIN' -ldl
for t in test_core test_layerwise test_jointq; do
  $CXX $FLAGS -o "$LIB/dropin_$t" "$REF/tests/test_main.cpp" "$REF/tests/$t.cpp" \
    -L"$LIB" -locw_dropin -locwg -Wl,-rpath,'$ORIGIN' -ldl
done
$CXX $FLAGS -O3 -pthread -o "$LIB/dropin_bench" "$HERE/dropin_bench.cpp" \
  -L"$LIB" -locw_dropin -locwg -Wl,-rpath,'$ORIGIN' -ldl
echo "build_dropin: built $LIB/{libocw_dropin.so,dropin_test_core,dropin_test_layerwise,dropin_test_jointq,dropin_bench}"
