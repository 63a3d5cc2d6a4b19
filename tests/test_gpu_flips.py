"""Trajectory differences between the B200 product and the CPU oracle are
rounding flips of a threshold decision, shown record by record.

Both libraries report, for every history record, the margins of the decisions
taken in that iteration (beig_result_margins): the converged-prefix test
(per_pair / tol of the pairs either side of the prefix, rr.cpp:35-36), the
warm-up shrink test (r / r_warm, strategy.cpp:49) and the slope test
((c_max - mu c) / (mu c), strategy.cpp:85), plus the termination test r / tol.
Where the (n_now, event, lock) trajectories first differ, one of these margins
must lie within rounding of its threshold — rounding measured as the two runs'
relative r_overall difference just before the split.  SD's
drop-threshold flips (K4 pivot decisions) are bounded in test_gpu_solvers.py.
"""
import numpy as np
import pytest

from tests.helpers import explain_divergence, first_divergence, laplacian_1d

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["si", "lobpcg", "tracemin"])
@pytest.mark.parametrize("strat", ["none", "fix", "slope", "slopek"])
@pytest.mark.parametrize("n", [100, 400])
def test_laplacian_divergence_is_a_rounding_flip(product, oracle, solver, strat, n):
    rp, col, val = laplacian_1d(n)
    tol = 1e-10
    out = []
    for L in (product, oracle):
        a = L.from_csr(n, rp, col, val)
        out.append(L.solve(a, solver, n_ev=4 if n == 100 else 10, seed=11, tol=tol,
                           strategy=L.strategy_config(strat)))
    g, o = out
    assert g.status == o.status
    np.testing.assert_allclose(g.values, o.values, rtol=1e-9)
    hg, ho = g.history, o.history
    i = first_divergence(hg, ho)
    if i is None:
        assert g.iterations == o.iterations
        return
    why = explain_divergence(hg, ho, g.margins, o.margins, i, tol)
    assert why is not None, (i, hg[i], ho[i], g.margins[i], o.margins[i])
    print(f"{solver}/{strat}/n={n}: records split at {i}: {why}")
