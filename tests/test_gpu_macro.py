"""Large-n paths of the GPU factorisation: macro panels (n > 4608 by default,
or OCWG_CHOL_MACRO) run the owner/worker tile Cholesky once per column panel
with a tcgen05 SYRK of the trailing matrix in between, and partial last tiles.

Checker: the reference's own sources compiled by oracle/build_ref.sh
(oracle/ref.py); the same tolerances as tests/test_gpu_parity.py.  At
n = 5000 the size-independent property is used instead: identity-H GPTQ is
RTN exactly (test_layerwise.cpp:47-63).
"""
import os

import numpy as np
import pytest

from tests.test_gpu_parity import g, prec, sym_close  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu


@pytest.fixture
def macro192():
    old = os.environ.get("OCWG_CHOL_MACRO")
    os.environ["OCWG_CHOL_MACRO"] = "192"  # 3 tiles per panel
    yield
    if old is None:
        del os.environ["OCWG_CHOL_MACRO"]
    else:
        os.environ["OCWG_CHOL_MACRO"] = old


def _gram(ref, n, seed):
    x = ref.random_gaussian(2 * n, n, seed)
    x[:, ::17] *= 20.0  # outlier channels
    return (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("n,act", [(700, True), (640, False)])
def test_macro_panel_factor(g, ref, prec, macro192, n, act):
    h = _gram(ref, n, 900 + n)
    order, hinv, u, damp = g.gptq_factor(h, act, 0.01)
    rhinv, ru, rdamp = ref.gptq_factor(h, act, 0.01)
    np.testing.assert_array_equal(order, ref.gptq_order(h, act))
    assert sym_close(hinv, rhinv) <= (1e-4 if prec == "fp32" else 1e-9)
    assert np.max(np.abs(u - ru)) <= (1e-4 if prec == "fp32" else 1e-9) * np.max(np.abs(ru))


def test_factor_odd_size_single_panel(g, ref):
    # nt = 65 with a 4-row last tile: the owner's last sub tile and the identity
    # padding of the last diagonal tile (no macro panels).  Checked against a
    # numpy fp64 restatement of layerwise.cpp:31-51 (the reference's own build
    # runs fixed-order loops under test: minutes at this size).
    n = 4100
    x = np.random.default_rng(4100).standard_normal((2 * n, n)).astype(np.float32)
    x[:, ::17] *= 20.0
    h = (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    order, hinv, u, damp = g.gptq_factor(h, True, 0.01)
    np.testing.assert_array_equal(order, ref.gptq_order(h, True))
    hd = h.astype(np.float64)
    lam = 0.01 * float(np.mean(np.diagonal(hd)))
    assert abs(damp - lam) <= 1e-12 * lam
    hp = hd[np.ix_(order, order)] + lam * np.eye(n)
    rhinv = np.linalg.inv(hp)
    assert sym_close(hinv, rhinv) <= 1e-4
    ru = np.linalg.cholesky(rhinv).T  # U = upper Cholesky factor of H_p^-1 (layerwise.cpp:47-51)
    assert np.max(np.abs(u - ru)) <= 1e-4 * np.max(np.abs(ru))


def test_macro_panel_gptq_codes(g, ref, macro192):
    n, m = 700, 256
    h = _gram(ref, n, 4242)
    w = ref.random_gaussian(n, m, 4243, 0.02)
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 128)
    q = g.gptq_quantize(w, h, cfg, g.GptqOptions(True, 0.01, 128), want_w_hat=True)
    rq = ref.gptq_quantize(w, h, 4, 1, 2, 128, True, 0.01, 128)
    match = float(np.mean(q.codes == rq[0]))
    assert match >= 0.999, match
    np.testing.assert_array_equal(q.scales, rq[1])
    np.testing.assert_array_equal(q.zeros, rq[2])


def test_large_n_identity_hessian_is_rtn(g, ref):
    # n > 4608: default macro panels (2048 columns), partial last tile (5000 % 64 = 8)
    n, m = 5000, 256
    w = ref.random_gaussian(n, m, 5000, 0.02)
    h = np.eye(n, dtype=np.float32) * 3.0
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 128)
    q = g.gptq_quantize(w, h, cfg, g.GptqOptions(True, 0.01, 128), want_w_hat=True)
    r = g.quantize_matrix(w, cfg)
    np.testing.assert_array_equal(q.codes, r.codes)
    np.testing.assert_array_equal(q.scales, r.scales)
    np.testing.assert_array_equal(q.w_hat, g.dequantize(q))
