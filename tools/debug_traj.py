"""Debug helper: compare product vs oracle trajectories on one scenario."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2409_05572_b200 import blockeig as B
from tests.helpers import laplacian_1d
P = B.Library('paper_2409_05572_b200/libblockeig_b200.so')
O = B.Library('oracle/_build/liborc_blockeig.so')
solver = sys.argv[1] if len(sys.argv) > 1 else 'sd'
strat = sys.argv[2] if len(sys.argv) > 2 else 'none'
n = 100
rp, col, val = laplacian_1d(n)
res = []
for L in (P, O):
    a = L.from_csr(n, rp, col, val)
    res.append(L.solve(a, solver, strategy=L.strategy_config(strat), n_ev=4, seed=11))
g, o = res
hg, ho = g.history, o.history
print('iters', g.iterations, o.iterations)
for i in range(0, min(len(hg), len(ho)), max(1, min(len(hg), len(ho)) // 40)):
    a, b = hg[i], ho[i]
    print(i + 1, f"{a['r_overall']:.6e} {b['r_overall']:.6e} rel={abs(a['r_overall']-b['r_overall'])/b['r_overall']:.2e}",
          a['n_now'], b['n_now'], a['event'], b['event'], a['rr_dim'], b['rr_dim'], a['ortho_flops'] - b['ortho_flops'])
