"""The CUDA sweep runs GPTQ in the closed form
    w_cur[k] = w[k] + sum_{i<k} G[k,i] (w[i] - w_hat[i]),
    G[k,i]   = L[n-1-i, n-1-k] / L[n-1-k, n-1-k],   L = chol(J hp J)
(paper_2603_28845_b200/csrc/factor.cu, sweep.cu) instead of the reference's
recurrence over U = chol(hp^-1)^T (layerwise.cpp:43-90).  These CPU tests pin
that restatement: in fp64 numpy it reproduces the reference's codes exactly
on seeded problems, and G equals V^-T - I with V = diag(U)^-1 U.
"""
import numpy as np
import pytest


def closed_form_gptq(orc, w, h, cfg, actorder, percdamp, block):
    """fp64 numpy restatement of the CUDA path's algorithm (test only)."""
    n, m = w.shape
    order = orc.gptq_order(h, actorder)
    hd = np.asarray(h, np.float32).astype(np.float64)
    damp = percdamp * float(np.mean(np.diagonal(hd)))
    hd[np.diag_indices_from(hd)] += damp
    hp = hd[np.ix_(order, order)]
    a = hp[::-1, ::-1]
    L = np.linalg.cholesky(a)
    Lr = L[::-1, ::-1]                       # Lr[k][i] = L[n-1-k][n-1-i] (upper)
    G = (Lr / np.diagonal(Lr)[None, :]).T    # G[k][i] = L[n-1-i][n-1-k] / L[n-1-k][n-1-k]
    G = np.tril(G, -1)
    grids = orc.calibrate_grids(w, cfg)
    gidx = orc.group_index_matrix(cfg, n, m)
    w0 = w[order].astype(np.float64)
    acc = np.zeros((n, m))
    delta = np.zeros((n, m))
    codes = np.zeros((n, m), np.int16)
    for ib in range(0, n, block):
        ie = min(n, ib + block)
        for i in range(ib, ie):
            orig = int(order[i])
            cur = (w0[i] + acc[i]).astype(np.float32)
            g = gidx[orig]
            code, w_hat = orc.quantize_scalar(cur, grids.scale[g], grids.zero[g], grids.qmin,
                                              grids.qmax)
            codes[orig] = code
            delta[i] = w0[i] - w_hat.astype(np.float64)
            acc[i + 1:ie] += np.outer(G[i + 1:ie, i], delta[i])
        acc[ie:] += G[ie:, ib:ie] @ delta[ib:ie]
    return codes, G, order, damp


@pytest.mark.parametrize("seed,n,m,actorder,block", [(1, 24, 40, True, 8), (2, 33, 17, False, 5),
                                                     (3, 64, 64, True, 16), (4, 48, 96, True, 48)])
def test_closed_form_reproduces_reference_codes(orc, seed, n, m, actorder, block):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((4 * n, n)).astype(np.float32)
    x[:, rng.choice(n, 2, replace=False)] *= 10
    h = (x.T.astype(np.float64) @ x).astype(np.float32)
    w = (0.02 * rng.standard_normal((n, m))).astype(np.float32)
    cfg = orc.QuantConfig(3, orc.Scheme.asymmetric, orc.Granularity.per_group, 8)
    ref = orc.gptq_quantize(w, h, cfg, orc.GptqOptions(actorder, 0.01, block))
    codes, _, _, _ = closed_form_gptq(orc, w, h, cfg, actorder, 0.01, block)
    assert float(np.mean(codes == ref.codes)) >= 0.999


def test_g_equals_unit_upper_inverse_transpose(orc):
    rng = np.random.default_rng(5)
    n = 40
    x = rng.standard_normal((200, n)).astype(np.float32)
    h = (x.T.astype(np.float64) @ x).astype(np.float32)
    order = orc.gptq_order(h, True)
    u, _, _ = orc.gptq_factor(h, order, 0.01)
    v = u / np.diagonal(u)[:, None]
    g_ref = np.linalg.inv(v).T - np.eye(n)
    _, g, _, _ = closed_form_gptq(orc, np.zeros((n, 1), np.float32), h,
                                  orc.QuantConfig(4, orc.Scheme.asymmetric,
                                                  orc.Granularity.per_channel, 128),
                                  True, 0.01, 8)
    np.testing.assert_allclose(g, g_ref, atol=1e-9)
