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
    # >= 65536 local rows: level 0 in the TMA format (offset dictionary, split views)
    ("poisson", 64, 2, {}),
    ("poisson", 72, 3, {}),
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


@pytest.mark.parametrize("n,nranks", [(32, 2), (64, 2), (40, 3)])
def test_split_passes_interior_ranges(n, nranks):
    """Each distributed pass runs its ghost-free interior rows while the halo
    exchange is in flight: the interior range must contain no
    row with a ghost column, and for z-slab partitions of a stencil it covers
    all but about one plane per neighbour (minus format alignment)."""
    p, c, v, f = synth.problem("poisson", n)
    multi = amgb.setup_dist(p, c, v, nranks=nranks, rank=-1, gather_below=1000, coarse_enough=100)
    for r in range(nranks):
        info = multi.dist_level_info(r, 0)
        ex = multi.dist_export(r, 0)
        nloc = info["row1"] - info["row0"]
        ap, ac, _ = ex["A"]
        a0, a1 = info["A_ib0"], info["A_ib1"]
        assert 0 <= a0 <= a1 <= nloc
        for i in range(a0, a1):
            assert np.all(ac[ap[i]:ap[i + 1]] < nloc), (r, i)
        nbr = (r > 0) + (r < nranks - 1)
        assert a1 - a0 >= nloc - nbr * n * n - 2 * 2048, (r, a0, a1, nloc)
        rp, rc, _ = ex["R"]
        b0, b1 = info["R_ib0"], info["R_ib1"]
        assert 0 <= b0 <= b1 <= info["crow1"] - info["crow0"]
        for i in range(b0, b1):
            assert np.all(rc[rp[i]:rp[i + 1]] < nloc)


def test_split_and_unsplit_passes_agree():
    import os
    p, c, v, f = synth.problem("poisson", 36)
    kw = dict(nranks=3, rank=-1, gather_below=600, coarse_enough=100)
    ms = amgb.setup_dist(p, c, v, **kw)
    os.environ["AMGB_NO_SPLIT"] = "1"
    try:
        mu = amgb.setup_dist(p, c, v, **kw)
    finally:
        del os.environ["AMGB_NO_SPLIT"]
    assert ms.dist_level_info(0, 0)["A_ib1"] > 0 and mu.dist_level_info(0, 0)["A_ib1"] == -1
    xs, its, rels, _ = ms.solve(dev(f), tol=1e-8)
    xu, itu, relu, _ = mu.solve(dev(f), tol=1e-8)
    assert its == itu
    a, b = host(xs), host(xu)
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    r = synth.random_vector(len(f))
    za, zb = host(ms.precond(dev(r))), host(mu.precond(dev(r)))
    assert np.array_equal(za, zb)  # no dots inside a V-cycle: bitwise


def test_weak_scaling_virtual_ranks_4_parts():
    """BASELINE configs[4] (C5) shape at a small size: Poisson on n x n x 4n
    (synth.weak_poisson: one n^3 z-slab per rank, h = 1/(n+1) everywhere),
    partitioned over 4 virtual ranks -- each rank's level-0 rows are exactly its
    slab -- against the single-GPU solve (iterations +-1, x within 1e-10 at equal
    count) and the oracle (iterations +-1, x within 1e-8)."""
    n, P = 24, 4
    p, c, v, f = synth.weak_poisson(P, n)
    assert len(f) == n * n * n * P
    kw = {"coarse_enough": 100}
    single = amgb.setup(p, c, v, **kw)
    multi = amgb.setup_dist(p, c, v, nranks=P, rank=-1, gather_below=500, **kw)
    st = multi.dist_info()["row_starts"]
    assert list(st) == [r * n ** 3 for r in range(P + 1)]  # one slab per rank
    xs, its, _, sts = single.solve(dev(f), tol=1e-8, maxiter=100)
    xm, itm, relm, stm = multi.solve(dev(f), tol=1e-8, maxiter=100)
    assert sts == stm == amgb.OK and abs(its - itm) <= 1 and relm <= 1.01e-8
    if its == itm:
        assert np.linalg.norm(host(xs) - host(xm)) <= 1e-10 * np.linalg.norm(host(xs))
    A = oracle.Csr(p, c, v)
    o = oracle.cg(A, f, tol=1e-8, maxiter=100, hier=oracle.Hierarchy(A, **kw))
    assert abs(itm - o["iters"]) <= 1
    if itm != o["iters"]:
        xm, itm, relm, stm = multi.solve(dev(f), tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(host(xm) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])
