"""QEP target correction on the GPU (ocwg_qep_target, layerwise.cpp:95-112)
against the reference's own qep_target / quantize_layer (oracle/_ref), on
seeded calibration pairs (x_fp, x_pert) whose statistics come from the
reference's accumulate_stats.  fp64 on both sides: the corrected target is
compared with rtol 1e-6; quantize_layer codes >= 99.9 % identical.  The
larger cases run several 128 x 128 DMMA tiles, the triangular k-range skip of
the L^-1 products and (n > 512) the macro-panel fp64 Cholesky."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2603_28845_b200 as pkg
    return pkg


def stats_pair(ref, n, t, seed):
    x = ref.random_gaussian(t, n, seed)
    xp = x + 0.05 * ref.random_gaussian(t, n, seed + 1)  # perturbed (quantized-upstream) inputs
    gram, cross = np.zeros((n, n)), np.zeros((n, n))
    ref.accumulate_stats(gram, cross, x, xp)
    return gram, cross


@pytest.mark.parametrize("n,m,alpha,eta", [(16, 24, 1.0, 0.01), (64, 40, 0.5, 0.05),
                                           (130, 70, 0.25, 0.01), (600, 300, 0.5, 0.01),
                                           (700, 260, 1.0, 0.02)])
def test_qep_target_matches_reference(g, ref, n, m, alpha, eta):
    gram, cross = stats_pair(ref, n, 4 * n, 900 + n)
    w = ref.random_gaussian(n, m, 77 + n, 0.02)
    want = ref.qep_target(w, gram, cross, alpha, eta)
    got = g.qep_target(w, g.CalibStats(gram, cross), g.QepOptions(alpha, eta))
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-9)


def test_qep_alpha_zero_is_identity_and_errors(g, ref):
    gram, cross = stats_pair(ref, 8, 32, 5)
    w = ref.random_gaussian(8, 5, 6)
    s = g.CalibStats(gram, cross)
    np.testing.assert_array_equal(g.qep_target(w, s, g.QepOptions(0.0, 0.01)), w)
    with pytest.raises(g.InvalidInput):
        g.qep_target(w, s, g.QepOptions(1.5, 0.01))
    with pytest.raises(g.InvalidInput):
        g.qep_target(w, s, g.QepOptions(0.5, 0.0))
    with pytest.raises(g.NumericError):  # zero gram: lambda = 0, LLT fails
        g.qep_target(w, g.CalibStats(np.zeros((8, 8)), cross), g.QepOptions(0.5, 0.01))


@pytest.mark.parametrize("method", ["rtn", "gptq"])
def test_quantize_layer_with_qep_matches_reference(g, ref, method):
    n, m = 64, 96
    gram, cross = stats_pair(ref, n, 256, 31)
    w = ref.random_gaussian(n, m, 32, 0.02)
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 32)
    opts = g.LayerQuantOptions(method, cfg, g.ScaleMode.minmax, g.GptqOptions(True, 0.01, 16),
                               g.QepOptions(0.7, 0.02))
    q = g.quantize_layer(w, g.CalibStats(gram, cross), opts)
    rc, rs, rz = ref.quantize_layer(w, gram, cross, method == "gptq", 4, 1, 2, 32, False, True,
                                    0.01, 16, (0.7, 0.02))
    assert float(np.mean(q.codes == rc)) >= 0.999
    np.testing.assert_array_equal(q.scales, rs)
    np.testing.assert_array_equal(q.zeros, rz)
