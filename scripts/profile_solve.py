"""Short solve driver for ncu captures: setup, one warm-up solve, one solve."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--problem", default="poisson")
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--relax", default="spai0")
ap.add_argument("--solver", default="cg")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
p, c, v, f = synth.problem(a.problem, a.n)
h = amgb.setup(p, c, v, {"precond.relax.type": a.relax, "solver.type": a.solver})
fd = torch.from_numpy(f).cuda()
if a.batch > 1:
    F = torch.stack([fd * (1.0 + 0.1 * j) for j in range(a.batch)])
    for i in range(a.solves):
        X, its, rels, st = h.solve_batched(F, tol=1e-8, maxiter=200)
        print(f"batched solve {i}: iters {list(its)} status {st}")
    sys.exit(0)
for i in range(a.solves):
    x, it, rel, st = h.solve(fd, tol=1e-8, maxiter=200)
    print(f"solve {i}: iters {it} rel {rel:.3e} status {st} launches {h.stats()['kernel_launches']}")
