"""The library's GEMM kernels (SIMT fp32/fp64 and tcgen05 3xTF32) against an
fp64 numpy product, over every operand-major combination the factorisation
and the GPTQ sweep use, including M/N/K tails and lower-triangle tiles."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 32), (200, 136, 64), (4032, 64, 64), (64, 520, 64), (300, 4096, 128),
          (1000, 1000, 100), (17, 33, 5)]


@pytest.fixture(scope="module")
def g():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2603_28845_b200 as pkg
    return pkg


@pytest.mark.parametrize("impl", [0, 1, 2], ids=["simt_fp32", "simt_fp64", "tc_tf32x3"])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("lower", [0, 1])
def test_gemm_accuracy(g, impl, ta, tb, lower):
    import torch
    rng = np.random.default_rng(1 + ta + 2 * tb + 4 * impl)
    dt = np.float64 if impl == 1 else np.float32
    for m, n, k in SHAPES:
        if lower and m != n:
            continue
        a = rng.standard_normal((k, m) if ta else (m, k)).astype(dt)
        b = rng.standard_normal((n, k) if tb else (k, n)).astype(dt)
        c = rng.standard_normal((m, n)).astype(dt)
        ref = 0.5 * c.astype(np.float64) - 1.5 * ((a.T if ta else a).astype(np.float64)
                                                   @ (b.T if tb else b).astype(np.float64))
        ad, bd, cd = (torch.from_numpy(v).cuda() for v in (a, b, c))
        ms = C.c_double()
        g._check(g.lib().ocwg_debug_gemm(g.context().handle, impl, m, n, k, -1.5, ad.data_ptr(),
                                         a.shape[1], ta, bd.data_ptr(), b.shape[1], tb, 0.5,
                                         cd.data_ptr(), n, lower, 1, C.byref(ms)))
        out = cd.cpu().numpy().astype(np.float64)
        if lower:  # only tiles touching the lower triangle are defined; check i >= j
            mask = np.tril(np.ones((m, n), bool))
            out, ref = out[mask], ref[mask]
        scale = np.sqrt(k) * 1.5 + 1
        tol = 1e-12 if impl == 1 else 1e-5
        err = float(np.max(np.abs(out - ref)) / scale)
        assert err <= tol, (impl, m, n, k, ta, tb, err)
