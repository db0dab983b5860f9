"""C-ABI boundary checks that need no GPU: libocwg.so loads, exports every
symbol include/ocwg.h declares, and its host-only entry points agree with the
reference (storage accounting, config validation).  Compute entry points on a
GPU-less host must fail loudly (no CPU fallback)."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ocwg.h"
LIB = ROOT / "paper_2603_28845_b200" / "lib" / "libocwg.so"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ocwg_[a-z0-9_]+)\s*\(", text)))


def test_library_built():
    assert LIB.exists(), "run __graft_entry__.build()"


def test_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (ocwg_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert len(declared_symbols()) >= 25


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_tcgen05_and_tma_in_sass():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass or "UTCMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass


def test_host_entry_points(ref):
    import paper_2603_28845_b200 as g
    assert g.lib().ocwg_version() == 1
    for bits in range(1, 9):
        for scheme in (0, 1):
            for gran in (0, 1, 2):
                cfg = g.QuantConfig(bits, g.Scheme(scheme), g.Granularity(gran), 3)
                for rows, cols in ((5, 7), (128, 128), (4096, 11008)):
                    assert g.uniform_storage_bytes(cfg, rows, cols) == ref.storage_bytes(
                        bits, scheme, gran, 3, rows, cols)
                    assert g.quant_group_count(cfg, rows, cols) == ref.group_count(
                        bits, scheme, gran, 3, rows, cols)
    assert g.uniform_storage_bytes(g.QuantConfig(4, g.Scheme.symmetric, g.Granularity.per_group, 128),
                                   128, 128) == 8448


def test_config_validation_matches_reference():
    import paper_2603_28845_b200 as g
    for bad in (g.QuantConfig(0), g.QuantConfig(9), g.QuantConfig(1, g.Scheme.symmetric),
                g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 0)):
        with pytest.raises(g.InvalidInput):
            g.validate_config(bad)
    g.validate_config(g.QuantConfig(1, g.Scheme.asymmetric))


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2603_28845_b200 as g
    with pytest.raises(g.CudaError):
        g.quantize_matrix(np.ones((4, 4), np.float32), g.QuantConfig())
