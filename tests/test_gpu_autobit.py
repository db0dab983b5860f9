"""AutoBit's candidate grid on the GPU (autobit.cpp:45-61 with
estimate_error :16-34) against the reference's own autobit.cpp compiled by
oracle/build_ref.sh.  Costs are exact; errors are fp64 sums in a different
order, so rtol 1e-10."""
import numpy as np
import pytest

from tests.test_gpu_parity import g  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols", [(64, 300), (257, 128), (33, 1000)])
@pytest.mark.parametrize("mode", ["naive", "act"])
def test_candidate_grid_matches_reference(g, ref, rows, cols, mode):
    w = ref.random_gaussian(rows, cols, 7 * rows + cols, 0.02)
    w[3, 5] = 0.4      # outlier
    w[7, :] = 0.0      # all-zero row: scale 1
    diag = np.linspace(0.25, 3.0, rows) if mode == "act" else None
    got = g.candidate_grid(w, mode, diag)
    rerr, rcost = ref.candidate_grid(w, 1 if mode == "act" else 0, diag)
    assert [c for _, c, _ in got] == [int(x) for x in rcost]
    np.testing.assert_allclose([e for _, _, e in got], rerr, rtol=1e-10, atol=0)
    assert [cfg.bits for cfg, _, _ in got] == [2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8]


def test_candidate_grid_errors(g, ref):
    w = ref.random_gaussian(8, 16, 1)
    with pytest.raises(g.InvalidInput):
        g.candidate_grid(w, "bogus")
    with pytest.raises(g.InvalidInput):
        g.candidate_grid(w, "act", np.ones(3))
    w[2, 2] = np.nan
    with pytest.raises(g.InvalidInput):
        g.candidate_grid(w)
