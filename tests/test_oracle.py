"""Pin the oracle (CPU only).

1. The reference's own hot-path tests (proj/tests/test_core.cpp,
   test_layerwise.cpp, and test_jointq.cpp for the f4 refiner), compiled
   unmodified against the oracle build, pass.
2. The numpy restatement agrees with the compiled reference on seeded inputs
   (bit-exact codes/grids/order; fp64-roundoff for U / H^-1 / stats).
3. The committed golden fixtures (tests/golden/, made by
   tests/golden/make_golden.py from the compiled reference) still reproduce.
"""
import itertools
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"


@pytest.mark.parametrize("name", ["ref_test_core", "ref_test_layerwise", "ref_test_jointq"])
def test_reference_unit_tests_pass_on_oracle_build(ref, name):
    exe = ROOT / "oracle" / "_ref" / name
    if not exe.exists():
        pytest.skip("reference test binaries not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


CFGS = list(itertools.product([2, 3, 4, 8], [0, 1], [0, 1, 2], [False, True]))


@pytest.mark.parametrize("bits,scheme,gran,mse", CFGS)
def test_numpy_rtn_matches_reference(ref, orc, bits, scheme, gran, mse):
    w = ref.random_gaussian(9, 37, 100 + bits * 7 + scheme * 3 + gran, 0.02)
    w[3, 5] *= 25.0  # an outlier
    group = 8
    rc, rs, rz = ref.quantize_matrix(w, bits, scheme, gran, group, mse)
    cfg = orc.QuantConfig(bits, orc.Scheme(scheme), orc.Granularity(gran), group)
    q = orc.quantize_matrix(w, cfg, orc.ScaleMode.mse_grid if mse else orc.ScaleMode.minmax)
    np.testing.assert_array_equal(q.codes, rc)
    np.testing.assert_array_equal(q.grids.scale.view(np.uint32), rs.view(np.uint32))
    np.testing.assert_array_equal(q.grids.zero, rz)
    d = orc.dequantize(q)
    np.testing.assert_array_equal(d, ref.dequantize(rc, rs, rz, bits, scheme, gran, group))


def test_degenerate_and_large_groups_match_reference(ref, orc):
    # constant groups (scale 1), all-zero groups, huge-magnitude constant groups
    w = np.zeros((4, 16), np.float32)
    w[1, :8] = 3.25
    w[2, :] = 1e6
    w[3, 8:] = -7.0
    w[3, 0] = 1e-30
    for scheme in (0, 1):
        rc, rs, rz = ref.quantize_matrix(w, 4, scheme, 2, 8)
        cfg = orc.QuantConfig(4, orc.Scheme(scheme), orc.Granularity.per_group, 8)
        q = orc.quantize_matrix(w, cfg)
        np.testing.assert_array_equal(q.codes, rc)
        np.testing.assert_array_equal(q.grids.scale, rs)
        np.testing.assert_array_equal(q.grids.zero, rz)


def test_fp16_quirk_restated(orc):
    # fp16.hpp's subnormal-half branch: 2e-5 encodes to
    # 0x00a8 and decodes to ~5.0068e-6 (IEEE binary16 would give ~2.0027e-5)
    assert int(orc.fp16_encode(np.float32(2e-5))) == 0xA8
    assert abs(float(orc.fp16_round(np.float32(2e-5))) - 5.0067901611328125e-06) < 1e-12
    for v in (0.0, 1.0, -1.0, 0.5, 2.0, 65504.0, 6.103515625e-05):
        assert float(orc.fp16_round(np.float32(v))) == v


def test_storage_bytes_known_answers(ref):
    # test_core.cpp:198-219
    assert ref.storage_bytes(4, 0, 2, 128, 128, 128) == 8448
    assert ref.storage_bytes(8, 0, 0, 0, 4, 4) == 18


@pytest.mark.parametrize("n,m,bits,scheme,gran,actorder,block", [
    (16, 12, 3, 0, 1, False, 32), (24, 40, 4, 1, 2, True, 8), (33, 17, 2, 1, 0, True, 5),
    (64, 64, 4, 1, 2, False, 32), (48, 80, 3, 0, 2, True, 16),
])
def test_numpy_gptq_matches_reference(ref, orc, n, m, bits, scheme, gran, actorder, block):
    w = ref.random_gaussian(n, m, 4000 + n, 0.02)
    x = ref.random_gaussian(4 * n, n, 5000 + m)
    h = (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    group = 8
    rc, rs, rz = ref.gptq_quantize(w, h, bits, scheme, gran, group, actorder, 0.01, block)
    cfg = orc.QuantConfig(bits, orc.Scheme(scheme), orc.Granularity(gran), group)
    q = orc.gptq_quantize(w, h, cfg, orc.GptqOptions(actorder, 0.01, block), return_debug=True)
    assert np.mean(q.codes == rc) >= 0.999
    np.testing.assert_array_equal(q.grids.scale, rs)
    np.testing.assert_array_equal(q.grids.zero, rz)
    np.testing.assert_array_equal(q.extra["order"], ref.gptq_order(h, actorder))
    hinv, u, damp = ref.gptq_factor(h, actorder, 0.01)
    assert abs(q.extra["damp"] - damp) <= 1e-12 * abs(damp)
    np.testing.assert_allclose(q.extra["u"], u, rtol=1e-9, atol=1e-12 * np.abs(u).max())
    np.testing.assert_allclose(q.extra["hinv"], hinv, rtol=1e-9, atol=1e-12 * np.abs(hinv).max())


def test_stats_streaming_matches_reference(ref, orc):
    a = ref.random_gaussian(30, 12, 22)
    b = ref.random_gaussian(30, 12, 23)
    gram, cross = np.zeros((12, 12)), np.zeros((12, 12))
    tc = ref.accumulate_stats(gram, cross, a, b)
    s = orc.CalibStats.zeros(12)
    orc.accumulate_stats(s, a, b)
    assert tc == 30 == s.token_count
    np.testing.assert_allclose(s.gram, gram, rtol=1e-12)
    np.testing.assert_allclose(s.cross, cross, rtol=1e-12, atol=1e-12)


def test_pack_roundtrip_exhaustive(orc, ref):
    # test_pipeline.cpp:93-114: payload length == storage_bytes, decode identical
    for bits in range(1, 9):
        for scheme in (0, 1):
            if scheme == 0 and bits < 2:
                continue
            for gran in (0, 1, 2):
                cfg = orc.QuantConfig(bits, orc.Scheme(scheme), orc.Granularity(gran), 3)
                w = ref.random_gaussian(5, 7, bits * 10 + gran)
                q = orc.quantize_matrix(w, cfg)
                p = orc.pack_uniform(q.codes, q.grids, cfg)
                assert len(p) == ref.storage_bytes(bits, scheme, gran, 3, 5, 7)
                q2 = orc.unpack_uniform(p, 5, 7, cfg)
                np.testing.assert_array_equal(orc.dequantize(q2), orc.dequantize(q))


def load_golden_case(ref, orc, g):
    """Regenerate a golden case's inputs from its seeds (reference generator)."""
    import hashlib
    bits, scheme, gran, group, actorder, block = (int(v) for v in g["cfg"])
    w = ref.random_gaussian(int(g["n"]), int(g["m"]), int(g["seed_w"]), float(g["sd_w"]))
    x = ref.random_gaussian(int(g["t"]), int(g["n"]), int(g["seed_x"]))
    if int(g["bf16"]):
        x = orc.bf16_round(x)
    gram, cross = np.zeros((x.shape[1],) * 2), np.zeros((x.shape[1],) * 2)
    ref.accumulate_stats(gram, cross, x, x)
    h = gram.astype(np.float32)
    assert hashlib.sha256(h.tobytes()).hexdigest() == str(g["h_sha256"])
    cfg = orc.QuantConfig(bits, orc.Scheme(scheme), orc.Granularity(gran), group)
    return w, x, h, cfg, bool(actorder), block


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.npz")), ids=lambda p: p.stem)
def test_golden_fixtures_reproduce(ref, orc, path):
    g = np.load(path)
    w, x, h, cfg, act, block = load_golden_case(ref, orc, g)
    bits, scheme, gran, group = cfg.bits, int(cfg.scheme), int(cfg.granularity), cfg.group_size
    rc, rs, rz = ref.gptq_quantize(w, h, bits, scheme, gran, group, act, 0.01, block)
    np.testing.assert_array_equal(rs, g["scales"])
    np.testing.assert_array_equal(rz, g["zeros"])
    grids = orc.Grids(rs, rz, orc.scheme_qmin(bits, cfg.scheme), orc.scheme_qmax(bits, cfg.scheme))
    assert orc.pack_uniform(rc, grids, cfg) == g["payload"].tobytes()
    np.testing.assert_array_equal(ref.gptq_order(h, act), g["order"])
    # numpy restatement against the same fixture (second opinion)
    q = orc.gptq_quantize(w, h, cfg, orc.GptqOptions(act, 0.01, block))
    assert np.mean(q.codes == rc) >= 0.999
    np.testing.assert_array_equal(q.grids.scale, rs)
