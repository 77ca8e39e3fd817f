"""Localise mismatches of the tiled update against the oracle (debug aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from _helpers import Restated as R, instance  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

rows, cols, k, tile = (int(x) for x in sys.argv[1:5])
m = instance(rows, cols, 1018191 / (26214 * 11314))
eng = P.Engine(P.InputMatrix(m), k)
f = P.init_factors(rows, cols, P.SolverConfig(rank=k))
eng.set_factors(f)
eng.precompute_h_products()
r, s = eng.get_product("r"), eng.get_product("s")
eng.update_h(P.SolverConfig(rank=k, tile_size=tile), P.Algorithm.tiled)
got = eng.get_factors().ht
want, _ = R.update_tiled(f.ht, s, r, tile, is_w=False)
bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
print("H mismatches:", len(bad), "of", got.size, "nonfinite:", (~np.isfinite(got)).sum())
if len(bad):
    print("rows:", np.unique(bad[:, 0])[:20], "cols:", np.unique(bad[:, 1])[:40])
    i, j = bad[0]
    print("first", i, j, got[i, j], want[i, j])
# W update from the updated state
eng.precompute_w_products()
p_, q_ = eng.get_product("p"), eng.get_product("q")
w0 = eng.get_factors().w
eng.update_w(P.SolverConfig(rank=k, tile_size=tile), P.Algorithm.tiled)
gw = eng.get_factors().w
ww, norms = R.update_tiled(w0, q_, p_, tile, is_w=True)
print("W nonfinite:", (~np.isfinite(gw)).sum(), "dev", np.abs(gw - ww).max() / np.abs(ww).max())
print("norms gpu", eng.get_product("column_norms")[:5], "oracle", norms[:5])
