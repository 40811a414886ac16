import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_05704_b200 as amgb, synth, oracle
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
p, c, v, f = synth.problem("poisson", 64)
md = amgb.setup_dist(p, c, v, nranks=2, rank=-1, gather_below=2000, coarse_enough=300, device=-1)
for rk in (0, 1):
    ex = md.dist_export(rk, 0)
    ap, ac, av = ex["A"]
    info = md.dist_level_info(rk, 0)
    nloc = info["row1"] - info["row0"]
    ng = info["ghosts"]
    n = nloc + ng
    ptr = np.concatenate([ap, ap[-1] + 1 + np.arange(ng, dtype=np.int64)])
    col = np.concatenate([ac, np.arange(nloc, n, dtype=np.int32)])
    val = np.concatenate([av, np.ones(ng)])
    x = synth.random_vector(n)
    yref = oracle.spmv(oracle.Csr(ptr, col, val), x)
    for env in ({}, {"AMGB_NO_DICT": "1"}):
        for k in list(os.environ):
            if k.startswith("AMGB_"): del os.environ[k]
        os.environ.update(env)
        h = amgb.setup(ptr, col, val, coarse_enough=300, dense_max=60000)
        y = h.level_op(0, amgb.OP_SPMV_A, x=dev(x), ny=n).cpu().numpy()
        err = np.abs(y - yref)
        bad = np.nonzero(err > 1e-12 * np.abs(yref).max())[0]
        print("rank", rk, env, "dict slices", h.level_info(0)["dict_slices_A"], "bad rows", len(bad), bad[:10], nloc)
