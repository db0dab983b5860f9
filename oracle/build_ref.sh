#!/usr/bin/env bash
# Builds the CPU oracle from the reference's OWN sources, unmodified, straight
# from the read-only tree (never copied into this repo):
#   /root/reference/proj/src/{matrix,quant,stats,layerwise}.cpp
# against our from-scratch Eigen-API shim (paper_2603_28845_b200/compat) and
# doctest shim (oracle/shim).  Outputs go to oracle/_ref/ only (git-ignored,
# travels to the GPU box with the snapshot):
#   oracle/_ref/libocw_ref.so        reference hot path + oracle/ref_capi.cpp C entry points
#   oracle/_ref/ref_test_core        proj/tests/test_core.cpp      (unmodified)
#   oracle/_ref/ref_test_layerwise   proj/tests/test_layerwise.cpp (unmodified)
# container.cpp / pipeline.cpp need nlohmann/json (absent) and are not built;
# the packer is restated in oracle/ocw_oracle.py (container.cpp:15-35,129-139).
set -euo pipefail
REF=${OCW_REFERENCE:-/root/reference/proj}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(dirname "$HERE")"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: $REF not present; skipping (prebuilt oracle/_ref is used if shipped)" >&2
  exit 0
fi
mkdir -p "$OUT"
CXX=${CXX:-g++}
FLAGS="-std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter -I$REF/include -I$ROOT/paper_2603_28845_b200/compat -I$HERE/shim"
SRCS="$REF/src/matrix.cpp $REF/src/quant.cpp $REF/src/stats.cpp $REF/src/layerwise.cpp"
# autobit.cpp (candidate_grid / estimate_error) uses std::function
# without including <functional>; it is force-included, the source is unmodified
$CXX $FLAGS -shared -o "$OUT/libocw_ref.so" $SRCS "$REF/src/autobit.cpp" "$REF/src/jointq.cpp" -include functional \
    "$HERE/ref_capi.cpp" -ldl
# container.cpp (OCW1 writer / parser) needs nlohmann/json: the
# image ships 3.11.3 inside cudnn_frontend; without it the container checker is
# skipped (tests that need it skip too)
JSON_DIR=${OCW_JSON_DIR:-$(python3 -c "import os, site; ps = [os.path.join(p, 'include/cudnn_frontend/thirdparty/nlohmann') for p in site.getsitepackages()]; print(next((p for p in ps if os.path.exists(os.path.join(p, 'json.hpp'))), ''))" 2>/dev/null)}
if [ -n "$JSON_DIR" ] && [ -f "$JSON_DIR/json.hpp" ]; then
  $CXX $FLAGS -I"$JSON_DIR" -include functional -shared -o "$OUT/libocw_ref_container.so" \
      "$REF/src/container.cpp" "$REF/src/matrix.cpp" "$REF/src/quant.cpp" \
      "$HERE/ref_out_of_path_stubs.cpp" "$HERE/ref_container_capi.cpp" -ldl
fi
for t in test_core test_layerwise; do
  $CXX $FLAGS -o "$OUT/ref_$t" "$REF/tests/test_main.cpp" "$REF/tests/$t.cpp" $SRCS -ldl
done
# jointq.cpp (the refiner of GPTQ output) and its own unit tests
$CXX $FLAGS -o "$OUT/ref_test_jointq" "$REF/tests/test_main.cpp" "$REF/tests/test_jointq.cpp" $SRCS \
    "$REF/src/jointq.cpp" -ldl
echo "build_ref: built $OUT/{libocw_ref.so,ref_test_core,ref_test_layerwise,ref_test_jointq}"
