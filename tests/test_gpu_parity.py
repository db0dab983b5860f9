"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Checker: the reference's own sources compiled by oracle/build_ref.sh
(oracle/ref.py) and the golden fixtures in tests/golden/.  Tolerances are the
north_star's (BASELINE.json):
  * integer codes: >= 99.9 % identical (observed: identical); order, grids,
    packing: bit-exact;
  * H and H^-1: |dH_ij| <= 1e-4 * sqrt(H_ii H_jj) (SURVEY §8(c) comparator);
  * relative reconstruction error sqrt(tr(D^T H D) / tr(W^T H W)) within 1e-3
    of the reference's value.
"""
import itertools
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"


@pytest.fixture(scope="module")
def g():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2603_28845_b200 as pkg
    return pkg


@pytest.fixture(params=["fp32", "fp64"])
def prec(g, request):
    """Factorisation + sweep arithmetic (fp32 default, fp64 reference class)."""
    g.set_precision(g.FP64 if request.param == "fp64" else g.FP32)
    yield request.param
    g.set_precision(g.FP32)


def sym_close(a, b, tol=1e-4):
    """|a_ij - b_ij| <= tol * sqrt(b_ii b_jj)."""
    d = np.sqrt(np.abs(np.outer(np.diagonal(b), np.diagonal(b))))
    return float(np.max(np.abs(a - b) / np.maximum(d, 1e-300)))


# ------------------------------------------------------------------ RTN / grids / packing
@pytest.mark.parametrize("bits,scheme,gran,mse",
                         list(itertools.product([2, 3, 4, 8], [0, 1], [0, 1, 2], [False, True])))
def test_rtn_bit_exact(g, ref, bits, scheme, gran, mse):
    w = ref.random_gaussian(33, 70, 300 + bits + 10 * scheme + 100 * gran, 0.02)
    w[5, 7] = 0.5  # outlier
    w[6, :] = 0.125  # constant row (degenerate groups)
    cfg = g.QuantConfig(bits, g.Scheme(scheme), g.Granularity(gran), 16)
    mode = g.ScaleMode.mse_grid if mse else g.ScaleMode.minmax
    q = g.quantize_matrix(w, cfg, mode)
    rc, rs, rz = ref.quantize_matrix(w, bits, scheme, gran, 16, mse)
    np.testing.assert_array_equal(q.codes, rc)
    np.testing.assert_array_equal(q.scales.view(np.uint32), rs.view(np.uint32))
    np.testing.assert_array_equal(q.zeros, rz)
    np.testing.assert_array_equal(g.dequantize(q), ref.dequantize(rc, rs, rz, bits, scheme, gran, 16))


def test_grids_large_magnitude_and_tiny_ranges(g, ref):
    w = np.zeros((6, 32), np.float32)
    w[0] = 1e6
    w[1, :16] = 3.0
    w[1, 16:] = np.linspace(-1e-9, 1e-9, 16)
    w[2] = np.linspace(-5, 5, 32)
    w[3, ::2] = 1e-30
    w[4] = -7.0
    w[5] = np.linspace(1000.0, 1000.0001, 32)
    for scheme in (0, 1):
        for mse in (False, True):
            cfg = g.QuantConfig(3, g.Scheme(scheme), g.Granularity.per_group, 16)
            q = g.quantize_matrix(w, cfg, g.ScaleMode.mse_grid if mse else g.ScaleMode.minmax)
            rc, rs, rz = ref.quantize_matrix(w, 3, scheme, 2, 16, mse)
            np.testing.assert_array_equal(q.codes, rc)
            np.testing.assert_array_equal(q.scales, rs)
            np.testing.assert_array_equal(q.zeros, rz)


def test_calibrate_errors(g):
    w = np.ones((4, 4), np.float32)
    w[1, 2] = np.nan
    with pytest.raises(g.InvalidInput):
        g.quantize_matrix(w, g.QuantConfig())
    with pytest.raises(g.InvalidInput):
        g.quantize_matrix(np.zeros((0, 4), np.float32), g.QuantConfig())


@pytest.mark.parametrize("bits", range(1, 9))
def test_pack_unpack_exhaustive(g, orc, ref, bits):
    # test_pipeline.cpp:93-114 + byte equality with the restated packer
    for scheme in (0, 1):
        if scheme == 0 and bits < 2:
            continue
        for gran in (0, 1, 2):
            for rows, cols in ((5, 7), (3, 1), (17, 129), (64, 256)):
                cfg = g.QuantConfig(bits, g.Scheme(scheme), g.Granularity(gran), 3)
                w = ref.random_gaussian(rows, cols, bits * 10 + gran + rows)
                q = g.quantize_matrix(w, cfg)
                p = g.pack_uniform(q)
                assert len(p) == ref.storage_bytes(bits, scheme, gran, 3, rows, cols)
                ocfg = orc.QuantConfig(bits, orc.Scheme(scheme), orc.Granularity(gran), 3)
                grids = orc.Grids(q.scales, q.zeros, q.qmin, q.qmax)
                assert p == orc.pack_uniform(q.codes, grids, ocfg)
                q2 = g.unpack_uniform(p, rows, cols, cfg)
                np.testing.assert_array_equal(q2.codes, q.codes)
                np.testing.assert_array_equal(g.dequantize(q2), g.dequantize(q))


# ------------------------------------------------------------------ order / factorisation
def test_order_bit_exact_with_ties(g, ref):
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 300, 2049):
        h = np.diag(rng.integers(0, 5, n).astype(np.float32))  # many ties
        for act in (False, True):
            np.testing.assert_array_equal(g.gptq_order(h, act), ref.gptq_order(h, act))
    h = np.zeros((2, 2), np.float32)
    h[0, 0], h[1, 1] = 1.0, 100.0  # test_layerwise.cpp:65-73
    assert list(g.gptq_order(h, True)) == [1, 0]
    assert list(g.gptq_order(h, False)) == [0, 1]


@pytest.mark.parametrize("n,act", [(8, False), (64, True), (200, True), (515, False)])
def test_factor_matches_reference(g, ref, prec, n, act):
    x = ref.random_gaussian(3 * n, n, 77 + n)
    x[:, ::13] *= 20.0  # outlier channels
    h = (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    order, hinv, u, damp = g.gptq_factor(h, act, 0.01)
    rhinv, ru, rdamp = ref.gptq_factor(h, act, 0.01)
    np.testing.assert_array_equal(order, ref.gptq_order(h, act))
    assert abs(damp - rdamp) <= 1e-12 * rdamp
    assert sym_close(hinv, rhinv) <= (1e-4 if prec == "fp32" else 1e-9)
    assert np.max(np.abs(u - ru)) <= (1e-4 if prec == "fp32" else 1e-9) * np.max(np.abs(ru))


def test_not_positive_definite_raises(g, ref, prec):
    # test_layerwise.cpp:119-128
    w = ref.random_gaussian(4, 4, 1)
    hneg = np.eye(4, dtype=np.float32)
    hneg[0, 0] = -100.0
    cfg = g.QuantConfig(4, g.Scheme.symmetric, g.Granularity.per_channel, 0)
    with pytest.raises(g.NumericError):
        g.gptq_quantize(w, hneg, cfg)
    x = ref.random_gaussian(12, 3, 2)
    with pytest.raises(g.InvalidInput):
        g.gptq_quantize(w, x.T @ x, cfg)
    with pytest.raises(g.InvalidInput):
        g.gptq_quantize(w, np.eye(4, dtype=np.float32), cfg, g.GptqOptions(percdamp=0.0))
    # numeric_error wins over a non-finite W (factorisation runs first, layerwise.cpp:43-60)
    wn = w.copy()
    wn[0, 0] = np.inf
    with pytest.raises(g.NumericError):
        g.gptq_quantize(wn, hneg, cfg)
    with pytest.raises(g.InvalidInput):
        g.gptq_quantize(wn, np.eye(4, dtype=np.float32), cfg)


# ------------------------------------------------------------------ GPTQ
def test_identity_hessian_reduces_to_rtn(g, ref, prec):
    # test_layerwise.cpp:47-63
    for seed in (1, 2, 3):
        w = ref.random_gaussian(8, 12, seed)
        h = (np.eye(8) * np.float32(3.7)).astype(np.float32)
        for gran in (0, 1, 2):
            cfg = g.QuantConfig(3, g.Scheme.symmetric, g.Granularity(gran), 4)
            a = g.gptq_quantize(w, h, cfg)
            b = g.quantize_matrix(w, cfg)
            np.testing.assert_array_equal(a.codes, b.codes)
            np.testing.assert_array_equal(a.scales, b.scales)
            np.testing.assert_array_equal(a.zeros, b.zeros)


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.npz")), ids=lambda p: p.stem)
def test_gptq_matches_golden(g, ref, orc, prec, path):
    from tests.test_oracle import load_golden_case
    gd = np.load(path)
    w, x, h, cfg_o, act, block = load_golden_case(ref, orc, gd)
    cfg = g.QuantConfig(cfg_o.bits, g.Scheme(int(cfg_o.scheme)), g.Granularity(int(cfg_o.granularity)),
                        cfg_o.group_size)
    q = g.gptq_quantize(w, h, cfg, g.GptqOptions(act, 0.01, block), want_w_hat=True)
    ref_q = g.unpack_uniform(gd["payload"].tobytes(), w.shape[0], w.shape[1], cfg)
    match = float(np.mean(q.codes == ref_q.codes))
    assert match >= 0.999, match
    np.testing.assert_array_equal(q.scales, gd["scales"])
    np.testing.assert_array_equal(q.zeros, gd["zeros"])
    if match == 1.0:
        assert g.pack_uniform(q) == gd["payload"].tobytes()
    np.testing.assert_array_equal(q.w_hat, g.dequantize(q))
    obj = ref.activation_objective(w, q.w_hat, h)
    obj0 = ref.activation_objective(w, np.zeros_like(w), h)
    assert abs(np.sqrt(obj / obj0) - float(gd["rel_err"])) <= 1e-3


def test_gptq_beats_rtn_almost_always(g, ref, prec):
    # test_layerwise.cpp:100-117 (pinned seeds, N <= 16)
    from oracle.ocw_oracle import Rng
    pick = Rng(31337)
    wins = 0
    for trial in range(200):
        n = 4 + pick.below(13)
        m = 1 + pick.below(16)
        bits = 2 + pick.below(3)
        w = ref.random_gaussian(n, m, 5000 + trial)
        x = ref.random_gaussian(2 * n, n, 6000 + trial)
        # correlated_gram = matmul(transpose(x), x) in fp32, k-ordered sums
        h = np.zeros((n, n), np.float32)
        for k in range(x.shape[0]):
            h += np.outer(x[k], x[k]).astype(np.float32)
        cfg = g.QuantConfig(bits, g.Scheme.symmetric, g.Granularity.per_channel, 0)
        og = g.activation_objective(w, g.dequantize(g.gptq_quantize(w, h, cfg)), h)
        orr = g.activation_objective(w, g.dequantize(g.quantize_matrix(w, cfg)), h)
        wins += og <= orr * (1 + 1e-9)
    assert wins >= 190


def test_activation_objective_matches_reference(g, ref):
    w = ref.random_gaussian(40, 24, 1, 0.02)
    wh = w + ref.random_gaussian(40, 24, 2, 0.001)
    x = ref.random_gaussian(100, 40, 3)
    h = (x.T @ x).astype(np.float32)
    a = g.activation_objective(w, wh, h)
    b = ref.activation_objective(w, wh, h)
    assert abs(a - b) <= 1e-10 * abs(b)


# ------------------------------------------------------------------ statistics
def test_accumulate_stats_streaming(g, ref, prec):
    # test_core.cpp:272-318, both arithmetic classes: fp64 SIMT (exact to
    # round-off) and the tensor-core path (bf16 parts, within the north_star's
    # 1e-4 H bar; the reference's own streaming test allows 1e-5 of max|gram|)
    a, b = ref.random_gaussian(3, 4, 22), ref.random_gaussian(6, 4, 23)
    ap, bp = ref.random_gaussian(3, 4, 24), ref.random_gaussian(6, 4, 25)
    two, one = g.CalibStats.zeros(4), g.CalibStats.zeros(4)
    g.accumulate_stats(two, a, ap)
    g.accumulate_stats(two, b, bp)
    g.accumulate_stats(one, np.vstack([a, b]), np.vstack([ap, bp]))
    assert np.max(np.abs(two.gram - one.gram)) <= 1e-5 * np.max(np.abs(one.gram))
    assert np.max(np.abs(two.cross - one.cross)) <= 1e-5 * max(1.0, np.max(np.abs(one.cross)))
    assert two.token_count == 9
    rg, rc = np.zeros((4, 4)), np.zeros((4, 4))
    ref.accumulate_stats(rg, rc, np.vstack([a, b]), np.vstack([ap, bp]))
    if prec == "fp64":
        np.testing.assert_allclose(one.gram, rg, rtol=1e-12)
        np.testing.assert_allclose(one.cross, rc, rtol=1e-12, atol=1e-12)
    else:
        assert sym_close(one.gram, rg) <= 2e-5, sym_close(one.gram, rg)
        assert np.max(np.abs(one.cross - rc)) <= 2e-5 * np.max(np.abs(rc))
    s = g.CalibStats.zeros(4)
    g.accumulate_stats(s, a, a)
    assert np.max(np.abs(s.cross)) == 0.0
    x = np.array([[1.0, 2.0, -1.0]], np.float32)
    s3 = g.CalibStats.zeros(3)
    g.accumulate_stats(s3, x, x)
    np.testing.assert_allclose(s3.gram, np.outer(x[0], x[0]).astype(np.float64))
    with pytest.raises(g.InvalidInput):
        g.accumulate_stats(g.CalibStats.zeros(4), ref.random_gaussian(2, 3, 1),
                           ref.random_gaussian(2, 3, 1))


@pytest.mark.parametrize("t,n,bf16_exact", [(3000, 520, False), (2500, 131, False),
                                            (4100, 264, True), (20000, 96, False),
                                            (131072, 128, False)])
def test_accumulate_stats_tensor_cores_vs_reference(g, ref, orc, t, n, bf16_exact):
    """accumulate_stats(stats, x_fp, x_hat) with X_hat != X through the
    tensor-core path (bf16-exact X_hat: one segment; general fp32: bf16
    parts), gram and cross against the reference's fp64 accumulate_stats
    (stats.cpp:10-19), streamed in two calls like the sweep driver may."""
    x = ref.random_gaussian(t, n, 1700 + n)
    x[:, 5] *= 20.0
    xh = x + 0.05 * ref.random_gaussian(t, n, 1800 + n)
    if bf16_exact:
        xh = orc.bf16_round(xh)
    s = g.CalibStats.zeros(n)
    k = t // 3
    g.accumulate_stats(s, x[:k], xh[:k])
    g.accumulate_stats(s, x[k:], xh[k:])
    rg, rc = np.zeros((n, n)), np.zeros((n, n))
    ref.accumulate_stats(rg, rc, x, xh)
    assert s.token_count == t
    eg = sym_close(s.gram, rg)
    d = np.sqrt(np.outer(np.diagonal(rg), np.diagonal(rg)))
    ec = float(np.max(np.abs(s.cross - rc) / d))
    print(f"accumulate_stats t={t} n={n}: gram {eg:.2e}, cross {ec:.2e} (of sqrt(H_ii H_jj))")
    assert eg <= 1e-4 and ec <= 1e-4, (eg, ec)
    np.testing.assert_array_equal(s.gram, s.gram.T)


@pytest.mark.parametrize("t,n", [(64, 64), (4096, 512), (1000, 520), (77, 136), (8192, 1024),
                                 (640, 264), (1500, 131), (300, 5)])
def test_hessian_tensor_core_vs_fp64(g, ref, orc, t, n):
    import torch
    x = orc.bf16_round(ref.random_gaussian(t, n, 900 + n))
    x[:, 3] *= 20.0
    x = orc.bf16_round(x)
    bits = orc.bf16_bits(x)
    h = g.hessian_bf16(bits)
    gram, cross = np.zeros((n, n)), np.zeros((n, n))
    ref.accumulate_stats(gram, cross, x, x)
    assert sym_close(h, gram) <= 1e-4, sym_close(h, gram)
    np.testing.assert_array_equal(h, h.T)
    # accumulate semantics
    h2 = g.hessian_bf16(bits, h)
    assert sym_close(h2, 2 * gram) <= 1e-4
    # SIMT cross-check kernel through the debug hook
    lib = g.lib()
    xd = torch.from_numpy(bits.view(np.int16)).cuda()
    hd = torch.zeros(n, n, dtype=torch.float32, device="cuda")
    g._check(lib.ocwg_debug_hessian_dev(g.context().handle, xd.data_ptr(), t, n, hd.data_ptr(), 0, 1))
    assert sym_close(hd.cpu().numpy(), gram) <= 1e-6


def test_quantize_layer_end_to_end_c1(g, ref, orc):
    """BASELINE config 1 end to end from calibration tokens (W + X -> codes,
    grids, W_hat, payload, H) against the reference golden fixture."""
    from tests.test_oracle import load_golden_case
    gd = np.load(GOLDEN / "c1_512x512_w4g128.npz")
    w, x, h_ref, _, _, _ = load_golden_case(ref, orc, gd)
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 128)
    q, payload, h = g.quantize_layer_x(w, orc.bf16_bits(x), cfg, g.GptqOptions(False, 0.01, 128))
    assert sym_close(h, h_ref) <= 1e-4
    ref_q = g.unpack_uniform(gd["payload"].tobytes(), 512, 512, cfg)
    match = float(np.mean(q.codes == ref_q.codes))
    assert match >= 0.999, match
    np.testing.assert_array_equal(q.scales, gd["scales"])
    assert len(payload) == 137216
    ocfg = orc.QuantConfig(4, orc.Scheme.asymmetric, orc.Granularity.per_group, 128)
    assert payload == orc.pack_uniform(q.codes, orc.Grids(q.scales, q.zeros, 0, 15), ocfg)
    obj = ref.activation_objective(w, q.w_hat, h_ref)
    obj0 = ref.activation_objective(w, np.zeros_like(w), h_ref)
    assert abs(np.sqrt(obj / obj0) - float(gd["rel_err"])) <= 1e-3


@pytest.mark.parametrize("bits,scheme", [(4, "asymmetric"), (3, "symmetric")])
def test_sweep_residual_division_equals_ieee(g, ref, monkeypatch, bits, scheme):
    # The 128-row chain divides by one residual step when every scale is in
    # [2^-40, 2^40] (always, for fp16 grids) and by the IEEE routine otherwise;
    # both are correctly rounded, so codes and W_hat agree bit for bit -- with
    # zeros, outliers and negative (symmetric) codes in the mix.
    n, m = 1024, 512
    x = ref.random_gaussian(2 * n, n, 77)
    x[:, ::13] *= 25.0
    h = (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    w = ref.random_gaussian(n, m, 78, 0.02)
    w[::7, ::5] = 0.0
    w[3, :] *= 400.0
    cfg = g.QuantConfig(bits, getattr(g.Scheme, scheme), g.Granularity.per_group, 128)
    opts = g.GptqOptions(True, 0.01, 128)
    q1 = g.gptq_quantize(w, h, cfg, opts, want_w_hat=True)
    monkeypatch.setenv("OCWG_SWEEP_EXACT_DIV", "1")
    q2 = g.gptq_quantize(w, h, cfg, opts, want_w_hat=True)
    np.testing.assert_array_equal(q1.codes, q2.codes)
    np.testing.assert_array_equal(q1.w_hat, q2.w_hat)
    if scheme == "symmetric":
        assert q1.codes.min() < 0


@pytest.mark.parametrize("n,m,t", [(131, 96, 1000), (37, 64, 300)])
def test_quantize_layer_x_unaligned_dim(g, ref, orc, n, m, t):
    """n % 8 != 0: the calibration rows are re-strided for TMA and still run on
    the tensor cores (no SIMT fallback); end to end against the reference."""
    w = ref.random_gaussian(n, m, 4000 + n, 0.02)
    x = orc.bf16_round(ref.random_gaussian(t, n, 4100 + n))
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 32)
    q, payload, h = g.quantize_layer_x(w, orc.bf16_bits(x), cfg, g.GptqOptions(True, 0.01, 128))
    gram, cross = np.zeros((n, n)), np.zeros((n, n))
    ref.accumulate_stats(gram, cross, x, x)
    assert sym_close(h, gram) <= 1e-4
    rc, rs, rz = ref.gptq_quantize(w, gram.astype(np.float32), 4, 1, 2, 32, True, 0.01, 128)
    assert float(np.mean(q.codes == rc)) >= 0.999
    np.testing.assert_array_equal(q.scales, rs)
    np.testing.assert_array_equal(q.zeros, rz)
    assert len(payload) == g.storage_bytes(q)


@pytest.mark.parametrize("t,n,ld,gsegs,csegs,f64,window", [
    (300, 64, 64, [(0, 0)], [], False, 0),
    (300, 64, 64, [(0, 0), (0, 1), (1, 0)], [], False, 0),
    (300, 64, 64, [(0, 0)], [(0, 2)], False, 0),
    (300, 64, 64, [(0, 0), (0, 1), (1, 0)], [(0, 2), (0, 3), (1, 2)], True, 0),
    (5000, 131, 136, [(0, 0), (0, 1), (1, 0)], [(0, 2), (0, 3), (1, 2)], True, 2048),
    (2000, 520, 520, [(1, 1)], [(3, 2)], False, 512),
])
def test_gram_kernel_segments(g, t, n, ld, gsegs, csegs, f64, window):
    """The general statistics kernel (gram_tc.cu) on random bf16 operands:
    every segment set against an fp64 numpy restatement of the same sum of
    products (stats.cpp:16-17 shape)."""
    import ctypes as C
    import torch
    rng = np.random.default_rng(t + n)
    ops = [torch.from_numpy((rng.standard_normal((t, ld)) * (1.0 if k < 2 else 0.05)).astype(np.float32))
           .to(torch.bfloat16).cuda() for k in range(4)]
    for o in ops:
        o[:, n:] = 0
    host = [o.float().cpu().numpy().astype(np.float64)[:, :n] for o in ops]
    want_g = sum(host[a].T @ host[b] for a, b in gsegs)
    want_c = sum(host[a].T @ host[b] for a, b in csegs) if csegs else None
    dt = torch.float64 if f64 else torch.float32
    gram = torch.zeros(n, n, dtype=dt, device="cuda")
    cross = torch.zeros(n, n, dtype=dt, device="cuda")
    arr = lambda v, t_: (t_ * max(1, len(v)))(*(v or [0]))  # noqa: E731
    opp = (C.c_void_p * 4)(*[o.data_ptr() for o in ops])
    lib = g.lib()
    g._check(lib.ocwg_debug_gram_dev(g.context().handle, C.cast(opp, C.c_void_p), 4, t, n, ld,
                                     len(gsegs), C.cast(arr([a for a, _ in gsegs], C.c_int), C.c_void_p),
                                     C.cast(arr([b for _, b in gsegs], C.c_int), C.c_void_p),
                                     len(csegs), C.cast(arr([a for a, _ in csegs], C.c_int), C.c_void_p),
                                     C.cast(arr([b for _, b in csegs], C.c_int), C.c_void_p),
                                     gram.data_ptr(), cross.data_ptr(), int(f64), 0, window))
    torch.cuda.synchronize()
    scale = np.sqrt(np.outer(np.abs(np.diagonal(host[0].T @ host[0])), np.abs(np.diagonal(host[0].T @ host[0]))))
    eg = float(np.max(np.abs(gram.double().cpu().numpy() - want_g) / scale))
    assert eg <= 2e-5, eg
    if want_c is not None:
        ec = float(np.max(np.abs(cross.double().cpu().numpy() - want_c) / scale))
        assert ec <= 2e-5, ec


def test_split_bf16_parts(g, orc):
    """fp32 statistics inputs -> bf16 parts (stats.cu): P1 = bf16(xp),
    P2 = bf16(xp - P1), D = fp64(xf) - fp64(xp), D1 = bf16(D), D2 = bf16(D - D1),
    pad columns zero, flags (1: xp not bf16-exact, 2: D != 0)."""
    import torch
    rng = np.random.default_rng(5)
    t, n, ld = 37, 13, 16
    xf = rng.standard_normal((t, n)).astype(np.float32)
    xp = (xf + 0.05 * rng.standard_normal((t, n))).astype(np.float32)
    dxp, dxf = torch.from_numpy(xp).cuda(), torch.from_numpy(xf).cuda()
    outs = [torch.zeros((t, ld), dtype=torch.int16, device="cuda") for _ in range(4)]
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    g._check(g.lib().ocwg_debug_split_dev(g.context().handle, dxp.data_ptr(), dxf.data_ptr(), t, n, ld,
                                          *[o.data_ptr() for o in outs], fl.data_ptr()))
    torch.cuda.synchronize()
    p1, p2, d1, d2 = [o.cpu().numpy().view(np.uint16) for o in outs]
    val = lambda b: (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    np.testing.assert_array_equal(p1[:, :n], orc.bf16_bits(xp))
    np.testing.assert_array_equal(p1[:, n:], 0)
    r = xp.astype(np.float64) - val(p1[:, :n])
    np.testing.assert_array_equal(p2[:, :n], orc.bf16_bits(r.astype(np.float32)))
    d = xf.astype(np.float64) - xp.astype(np.float64)
    np.testing.assert_array_equal(d1[:, :n], orc.bf16_bits(d.astype(np.float32)))
    assert int(fl.item()) == 3


@pytest.mark.gpu
def test_column_major_statistics_layout(ref):
    """ocwg_set_stats_layout(OCWG_COL_MAJOR) (the drop-in's CalibStats storage):
    gram / cross in and out column-major give the transposes of the row-major
    results (quantize_layer / qep_target through the column-major drop-in are
    covered by the reference's own tests in test_gpu_dropin.py)."""
    import ctypes as C

    import paper_2603_28845_b200 as g
    lib = g.lib()
    n, t = 72, 300
    xp = ref.random_gaussian(t, n, 4401)
    xf = xp + 0.05 * ref.random_gaussian(t, n, 4402)
    g0 = ref.random_gaussian(n, n, 4403).astype(np.float64)
    g0 = g0 + g0.T  # the accumulated gram is symmetric; cross need not be
    c0 = ref.random_gaussian(n, n, 4404).astype(np.float64)
    out = {}
    for layout in (0, 1):
        h = C.c_void_p()
        assert lib.ocwg_create(0, C.byref(h)) == 0
        try:
            assert lib.ocwg_set_stats_layout(h, layout) == 0
            gm = np.ascontiguousarray(g0 if layout == 0 else g0.T).copy()
            cm = np.ascontiguousarray(c0 if layout == 0 else c0.T).copy()
            tc = C.c_uint64(0)
            assert lib.ocwg_accumulate_stats(h, xf.ctypes.data, xp.ctypes.data, t, n, gm.ctypes.data,
                                             cm.ctypes.data, C.byref(tc)) == 0
            out[layout] = (gm, cm)
        finally:
            lib.ocwg_destroy(h)
    np.testing.assert_array_equal(out[1][0], out[0][0].T)
    np.testing.assert_array_equal(out[1][1], out[0][1].T)
    assert lib.ocwg_set_stats_layout(g.context().handle, 7) == 1  # invalid layout
