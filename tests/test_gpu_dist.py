"""The row-partitioned (multi-GPU) solve path on ONE GPU: "virtual ranks"
(amg_setup_dist with rank = -1) run every rank's kernels, halo exchanges (as
device copies), all-reduces and the coarse-level all-gather of the NCCL path in
one process.  Results must match the single-GPU path (same hierarchy; row sums
in the same order, only dot-product summation order differs) and the oracle.
GPU only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


CASES = [
    ("poisson", 32, 2, {}),
    ("poisson", 32, 4, {}),
    ("poisson_perm", 24, 3, {}),
    ("varcoef", 24, 2, {"relax": "chebyshev"}),
    ("convdiff", 20, 3, {"relax": "damped_jacobi", "solver": "bicgstab"}),
    ("poisson", 25, 2, {"npre": 2, "npost": 2}),
]


@pytest.mark.parametrize("gen,n,nranks,kw", CASES)
def test_virtual_ranks_match_single_gpu_and_oracle(gen, n, nranks, kw):
    p, c, v, f = synth.problem(gen, n)
    kw = dict(kw, coarse_enough=100)
    single = amgb.setup(p, c, v, **kw)
    multi = amgb.setup_dist(p, c, v, nranks=nranks, rank=-1, gather_below=500, **kw)
    di = multi.dist_info()
    assert di["nranks"] == nranks and di["first_replicated"] >= 1
    maxiter = 200
    xs, its, rels, sts = single.solve(dev(f), tol=1e-8, maxiter=maxiter)
    xm, itm, relm, stm = multi.solve(dev(f), tol=1e-8, maxiter=maxiter)
    assert sts == stm == amgb.OK
    assert abs(its - itm) <= 1, (its, itm)
    assert relm <= 1.01e-8
    if its == itm:
        a, b = host(xs), host(xm)
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)
    # the oracle, iterations +-1 and x at equal count
    A = oracle.Csr(p, c, v)
    okw = {k: val for k, val in kw.items() if k not in ("solver",)}
    hier = oracle.Hierarchy(A, **okw)
    fn = oracle.bicgstab if kw.get("solver") == "bicgstab" else oracle.cg
    o = fn(A, f, tol=1e-8, maxiter=maxiter, hier=hier)
    assert abs(itm - o["iters"]) <= 1
    if itm != o["iters"]:
        xm, itm, relm, stm = multi.solve(dev(f), tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(host(xm) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


@pytest.mark.parametrize("nranks", [2, 3])
def test_virtual_ranks_vcycle(nranks):
    p, c, v, f = synth.problem("poisson_perm", 22)
    single = amgb.setup(p, c, v, coarse_enough=100)
    multi = amgb.setup_dist(p, c, v, nranks=nranks, rank=-1, gather_below=400, coarse_enough=100)
    r = synth.random_vector(len(f))
    zs = host(single.precond(dev(r)))
    zm = host(multi.precond(dev(r)))
    assert np.linalg.norm(zs - zm) <= 1e-13 * np.linalg.norm(zs)
    zo = oracle.Hierarchy(oracle.Csr(p, c, v), coarse_enough=100).precond(r)
    assert np.linalg.norm(zm - zo) <= 1e-12 * np.linalg.norm(zo)


def test_virtual_ranks_zero_rhs_and_host_path():
    p, c, v, f = synth.problem("poisson", 20)
    multi = amgb.setup_dist(p, c, v, nranks=2, rank=-1, gather_below=300, coarse_enough=60)
    x, it, rel, st = multi.solve(dev(np.zeros_like(f)), x=dev(np.ones_like(f)))
    assert it == 0 and st == amgb.OK and np.all(host(x) == 0)
    xh, it, rel, st = multi.solve_host(f, tol=1e-8)
    single = amgb.setup(p, c, v, coarse_enough=60)
    xs, its, _, _ = single.solve(dev(f), tol=1e-8)
    assert it == its and np.linalg.norm(xh - host(xs)) <= 1e-10 * np.linalg.norm(xh)


def test_nccl_transport_selftest():
    """The NCCL entry points (dlopen) with the executor's argument order, directly
    and inside a captured CUDA graph, on a 1-rank communicator."""
    import torch as _t
    _t.cuda.init()
    amgb.nccl_selftest(0)
