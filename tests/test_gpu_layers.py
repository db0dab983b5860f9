"""Layers sharing one calibration input (the sweep driver's
q/k/v and gate/up groups, run_layerwise_sweep pipeline.cpp:215-226): one
Hessian and one factorisation for all of them must give, for every W, exactly
the result of a separate quantize_layer_x call (codes, grids, payload)."""
import numpy as np
import pytest

from tests.test_gpu_parity import g  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def test_shared_input_layers_equal_separate_calls(g, ref, orc):
    n, t = 512, 4096
    x = orc.bf16_bits(ref.random_gaussian(t, n, 71))
    ws = [ref.random_gaussian(n, mm, 72 + i, 0.02) for i, mm in enumerate((512, 384, 1024))]
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 128)
    opts = g.GptqOptions(True, 0.01, 128)
    res = g.quantize_layers_x(ws, x, cfg, opts)
    assert len(res) == 3
    for w, (q, payload) in zip(ws, res):
        q1, p1, _h = g.quantize_layer_x(w, x, cfg, opts)
        np.testing.assert_array_equal(q.codes, q1.codes)
        np.testing.assert_array_equal(q.scales, q1.scales)
        np.testing.assert_array_equal(q.zeros, q1.zeros)
        assert payload == p1
        assert payload == g.pack_uniform(q)


def test_shared_input_layers_errors(g, ref, orc):
    x = orc.bf16_bits(ref.random_gaussian(64, 32, 1))
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 16)
    with pytest.raises(g.InvalidInput):
        g.quantize_layers_x([], x, cfg, g.GptqOptions())
    with pytest.raises(g.InvalidInput):
        g.quantize_layers_x([np.zeros((16, 8), np.float32)], x, cfg, g.GptqOptions())
