"""Two ocwg contexts on two GPUs in ONE process (kernel
function attributes and the SM count are per device, so the second device's
>48 KB shared-memory kernels must not depend on what the first device set).
The same layer through device 0 and device 1 must give identical codes, grids
and payload.  Skipped on a box with a single GPU."""
import numpy as np
import pytest

from tests.test_gpu_parity import g  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def test_second_device_in_same_process(g, ref, orc):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs in one process")
    n, m, t = 640, 512, 4096
    x = orc.bf16_bits(ref.random_gaussian(t, n, 91))
    w = ref.random_gaussian(n, m, 92, 0.02)
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 128)
    opts = g.GptqOptions(True, 0.01, 128)
    q0, p0, h0 = g.quantize_layer_x(w, x, cfg, opts, device=0)
    q1, p1, h1 = g.quantize_layer_x(w, x, cfg, opts, device=1)
    np.testing.assert_array_equal(q0.codes, q1.codes)
    np.testing.assert_array_equal(q0.scales, q1.scales)
    np.testing.assert_array_equal(q0.zeros, q1.zeros)
    assert p0 == p1
    if h0 is not None and h1 is not None:
        np.testing.assert_array_equal(h0, h1)
    # and device 0 again after device 1 ran (the attributes are set per launch)
    q2, p2, _ = g.quantize_layer_x(w, x, cfg, opts, device=0)
    np.testing.assert_array_equal(q0.codes, q2.codes)
    assert p0 == p2
