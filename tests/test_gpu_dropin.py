"""The reference's OWN unit tests (proj/tests/test_core.cpp, test_layerwise.cpp,
test_jointq.cpp,
compiled unmodified by paper_2603_28845_b200/cpp/build_dropin.sh) linked
against the C++ drop-in (ocw:: interface over libocwg.so) instead of the
reference's src/{quant,stats,layerwise}.cpp -- every known-answer, exact-
equivalence, statistical and error-contract test of the hot path, run on the
GPU implementation."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2603_28845_b200" / "lib"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dropin_test_core", "dropin_test_layerwise",
                                  "dropin_test_jointq"])
def test_reference_unit_tests_pass_on_gpu_dropin(name):
    exe = LIB / name
    if not exe.exists():
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OCW_SHIM_NO_BLAS": "1"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_dropin_exports_reference_interface():
    so = LIB / "libocw_dropin.so"
    if not so.exists():
        pytest.skip("drop-in not built")
    syms = subprocess.run(["nm", "-D", "-C", "--defined-only", str(so)], capture_output=True,
                          text=True).stdout
    for fn in ["ocw::gptq_quantize(", "ocw::quantize_layer(", "ocw::accumulate_stats(",
               "ocw::gptq_order(", "ocw::calibrate_grids(", "ocw::quantize_matrix(",
               "ocw::dequantize(", "ocw::qep_target(", "ocw::activation_objective(",
               "ocw::jointq_refine(", "ocw::jointq_objective(",
               "ocw::jointq_optimal_group_scale("]:
        assert fn in syms, fn
    libs = subprocess.run(["ldd", str(so)], capture_output=True, text=True).stdout
    assert "libocwg.so" in libs
