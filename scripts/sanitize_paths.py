"""Small runs of every device path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): GPU setup incl. device aggregation, TMA (dictionary, value
index), TMA-CSR, SELL (8- and 16-bit value index), row-block CSR, the fused level
ops, batched, mixed precision, BiCGStab / GMRES / IDR(s), Chebyshev, virtual ranks
(split passes), host formats."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()  # noqa: E731
# TMA + dictionary level 0 (>= 65536 rows), GPU setup + device formats
p, c, v, f = synth.problem("poisson", 41)
h = amgb.setup(p, c, v, coarse_enough=300)
x, it, rel, st = h.solve(dev(f), tol=1e-8)
print("cg", it, rel, st)
X, its, rels, st = h.solve_batched(torch.stack([dev(f)] * 4), tol=1e-8)
print("batched4", list(its), st)
X, its, rels, st = h.solve_batched(torch.stack([dev(f)] * 8), tol=1e-8)
print("batched8", list(its), st)
hm = amgb.setup(p, c, v, coarse_enough=300, precision="mixed")
print("mixed", hm.solve(dev(f), tol=1e-8)[1:])
# the fused production kernels one launch each (amg_level_op_ex)
n0 = len(f)
fv = dev(np.linspace(1.0, 2.0, n0))
y, y2, y3 = (torch.empty(n0, dtype=torch.float64, device="cuda") for _ in range(3))
h.level_op_ex(0, amgb.OP_RES0, in0=fv, out0=y)
h.level_op_ex(0, amgb.OP_RELAX_RHO, in0=fv, in1=fv, out0=y)
h.level_op_ex(0, amgb.OP_CG_DIR, in0=fv, in1=fv, out0=y, out1=y2, scalar=0.5)
h.level_op_ex(0, amgb.OP_CG_UPDATE, in0=fv, in1=fv, out0=y, out1=y2, out2=y3, scalar=0.5)
print("level ops", h.level_info(0)["formats"])
# every format forced: TMA-CSR everywhere, SELL everywhere (16-bit value indices on level 1)
for fmt in ("tmacsr", "sell", "tma"):
    os.environ["AMGB_FORMAT"] = fmt
    hf = amgb.setup(p, c, v, coarse_enough=300)
    print(fmt, hf.solve(dev(f), tol=1e-8)[1:], [hf.level_info(l)["formats"] for l in range(hf.nlevels)])
os.environ.pop("AMGB_FORMAT")
os.environ["AMGB_VIDX"] = "0"  # the fp64-array stores
print("fp64 arrays", amgb.setup(p, c, v, coarse_enough=300).solve(dev(f), tol=1e-8)[1:])
os.environ.pop("AMGB_VIDX")
# non-symmetric: BiCGStab, GMRES, IDR(s)
p2, c2, v2, f2 = synth.problem("convdiff", 16)
for solver, extra in (("bicgstab", {}), ("gmres", {}), ("idrs", {"idrs_s": 4})):
    hs = amgb.setup(p2, c2, v2, solver=solver, coarse_enough=200, relax="damped_jacobi", **extra)
    print(solver, hs.solve(dev(f2), tol=1e-8)[1:])
# Chebyshev
p3, c3, v3, f3 = synth.problem("varcoef", 20)
print("cheb", amgb.setup(p3, c3, v3, relax="chebyshev", coarse_enough=200).solve(dev(f3), tol=1e-8)[1:])
# virtual ranks: split passes on TMA level 0 (64^3 / 2 ranks)
p4, c4, v4, f4 = synth.problem("poisson", 64)
md = amgb.setup_dist(p4, c4, v4, nranks=2, rank=-1, gather_below=2000, coarse_enough=300)
print("dist", md.solve(dev(f4), tol=1e-8)[1:], md.dist_level_info(0, 0)["A_ib1"])
# permuted (explicit TMA slices), host formats
os.environ["AMGB_HOST_CONVERT"] = "1"
p5, c5, v5, f5 = synth.problem("poisson_perm", 40)
print("perm", amgb.setup(p5, c5, v5, coarse_enough=300).solve(dev(f5), tol=1e-8)[1:])
