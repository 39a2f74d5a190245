import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2412_12506_b200 as g
from tests import cases as K
from oracle import ref
ctx = g.Context(0)
spec, cfg = K.baseline_configs()["C3-SAI"]
R = ref.RefMultigrid(spec, cfg)
mg = g.Multigrid(ctx, cfg, g.Problem(spec, min_depth=cfg.min_depth))
got = mg.estimate_eta(kind=g._lib.KRYLOV_GMRES, seed=0)
want = R.eta(kind=1, seed=0)
print("got", got["iterations"], got["residuals"][:5], got["residuals"][-3:])
print("want", want["iterations"], want["residuals"][:5], want["residuals"][-3:])
for l in range(R.depth - 1):
    Bg = mg.smoother(l).sai_matrix(); Br = R.sai_matrix(l)
    st = mg.smoother(l).sai_stats()
    d = np.abs(Bg[2] - Br[2]).max(); nrm = np.abs(Br[2]).max()
    print("level", l, "B maxdiff", d, "rel", d / nrm, "ls", st.ls_dims(), "def", st.rank_deficient_columns)
