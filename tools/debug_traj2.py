"""Debug helper: iteration-by-iteration record diff over a window."""
import sys
sys.path.insert(0, '.')
from paper_2409_05572_b200 import blockeig as B
from tests.helpers import laplacian_1d
P = B.Library('paper_2409_05572_b200/libblockeig_b200.so')
O = B.Library('oracle/_build/liborc_blockeig.so')
solver, strat, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
n = 100
rp, col, val = laplacian_1d(n)
res = []
for L in (P, O):
    a = L.from_csr(n, rp, col, val)
    res.append(L.solve(a, solver, strategy=L.strategy_config(strat), n_ev=4, seed=11))
hg, ho = res[0].history, res[1].history
prev = [0, 0]
for i in range(lo, hi):
    a, b = hg[i], ho[i]
    print(a['iteration'], f"{a['r_overall']:.10e} {b['r_overall']:.10e}", 'n', a['n_now'], b['n_now'], 'ev', a['event'], b['event'],
          'lock', a['lock_count'], b['lock_count'], 'd', a['rr_dim'], b['rr_dim'],
          'dortho', a['ortho_flops'] - prev[0], b['ortho_flops'] - prev[1], 'spmv', a['spmv_cols'], b['spmv_cols'])
    prev = [a['ortho_flops'], b['ortho_flops']]
