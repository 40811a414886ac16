import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_05704_b200 as amgb, synth
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p, c, v, f = synth.problem("poisson", n)
single = amgb.setup(p, c, v, coarse_enough=300)
print("single", single.solve(dev(f), tol=1e-8)[1:])
r = synth.random_vector(len(f))
zs = single.precond(dev(r)).cpu().numpy()
for env in ({}, {"AMGB_HOST_CONVERT": "1"}, {"AMGB_NO_DICT": "1"}):
    for k in list(os.environ):
        if k.startswith("AMGB_"): del os.environ[k]
    os.environ.update(env)
    md = amgb.setup_dist(p, c, v, nranks=int(os.environ.get("NR", "2")) if False else 2, rank=-1, gather_below=2000,
                         coarse_enough=300)
    for rk in range(2):
        ex = md.dist_export(rk, 0)
        ap, ac, av = ex["A"]
        nloc = md.dist_level_info(rk, 0)["row1"] - md.dist_level_info(rk, 0)["row0"]
        rows = [i for i in range(0, nloc, 32) if i + 32 <= nloc]
        bad = 0
        for s0 in rows[:5000]:
            offs = set()
            w = 0
            for i in range(s0, s0 + 32):
                cc = ac[ap[i]:ap[i + 1]]
                w = max(w, len(cc))
                offs.update((cc.astype(np.int64) - i).tolist())
            if len(offs) == w and any(o > 0 and o >= nloc - s0 for o in offs):
                bad += 1
        print("rank", rk, "uniform slices with ghost offsets", bad, "level0 info", md.level_info(0)["dict_slices_A"])
    zm = md.precond(dev(r)).cpu().numpy()
    y0 = md.level_op(0, amgb.OP_SPMV_A, x=dev(r), ny=len(f)).cpu().numpy() if False else None
    print(env, "solve", md.solve(dev(f), tol=1e-8)[1:], "precond rel diff", np.linalg.norm(zm - zs) / np.linalg.norm(zs))
