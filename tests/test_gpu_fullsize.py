"""BASELINE.json configurations at FULL size against the oracle (GPU only).

* configs[2] (256^3 variable-coefficient Poisson, Chebyshev smoother): one
  preconditioner application z = M r on the full hierarchy, element by element
  against the oracle's V-cycle (1e-12 relative), and the converged solve checked
  through its true residual computed by the oracle's SpMV.
* configs[3] (200^3 convection-diffusion, BiCGStab + damped Jacobi): the whole
  solve against the oracle's (iterations +-1; x within 1e-8 at equal count).
* the headline (BASELINE.json metric, 256^3 Poisson CG + SA/SPAI-0): the whole
  solve against the oracle's, and every row of the level-0/1 fused passes.
(configs[0] and configs[1] at full size: tests/test_gpu_parity.py; bench.py also
repeats the headline parity check on every bench run: parity_full_size.)"""
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


def test_config2_varcoef256_chebyshev_full_size():
    p, c, v, f = synth.problem("varcoef", 256)
    h = amgb.setup(p, c, v, relax="chebyshev")
    A = oracle.Csr(p, c, v)
    ho = oracle.Hierarchy(A, relax="chebyshev")
    assert h.nlevels == ho.nlevels
    r = synth.random_vector(len(f))
    z = host(h.precond(dev(r)))
    zo = ho.precond(r)
    assert np.linalg.norm(z - zo) <= 1e-12 * np.linalg.norm(zo)
    x, it, rel, st = h.solve(dev(f), tol=1e-8, maxiter=100)
    assert st == amgb.OK
    res = f - oracle.spmv(A, host(x))
    assert np.linalg.norm(res) <= 1.01e-8 * np.linalg.norm(f)


def test_config3_convdiff200_bicgstab_full_size():
    p, c, v, f = synth.problem("convdiff", 200)
    kw = {"relax": "damped_jacobi"}
    h = amgb.setup(p, c, v, solver="bicgstab", **kw)
    A = oracle.Csr(p, c, v)
    ho = oracle.Hierarchy(A, **kw)
    x, it, rel, st = h.solve(dev(f), tol=1e-8, maxiter=100)
    o = oracle.bicgstab(A, f, tol=1e-8, maxiter=100, hier=ho)
    assert st == amgb.OK and o["status"] == 0
    assert abs(it - o["iters"]) <= 1, (it, o["iters"])
    if it != o["iters"]:
        x, it, rel, st = h.solve(dev(f), tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(host(x) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


def test_headline_h0_poisson256_full_size():
    """The headline configuration (BASELINE.json metric: 256^3 Poisson, CG +
    SA/SPAI-0 to 1e-8) through the production path (device-side loop, TMA /
    SELL store), against a full oracle solve: iterations +-1 and x within 1e-8
    at equal count (north star); then every row of the level-0 and level-1
    fused passes (the a1 / a5 / a6 kernels of bench.py's step) against the
    oracle under the a-priori bound of tests/test_gpu_formats.py."""
    from test_gpu_formats import U, check_rows, dot_bound, row_bound

    p, c, v, f = synth.problem("poisson", 256)
    h = amgb.setup(p, c, v)
    assert h.level_info(0)["fmt_A"] == amgb.FMT_TMA and h.level_info(0)["dict_slices_A"] > 0
    assert h.level_info(0)["fmt_P"] == amgb.FMT_TMACSR
    A = oracle.Csr(p, c, v)
    ho = oracle.Hierarchy(A)
    assert h.nlevels == ho.nlevels
    x, it, rel, st = h.solve(dev(f), tol=1e-8, maxiter=100)
    o = oracle.cg(A, f, tol=1e-8, maxiter=100, hier=ho)
    assert st == amgb.OK and o["status"] == 0
    assert abs(it - o["iters"]) <= 1, (it, o["iters"])
    if it != o["iters"]:
        x, it, rel, st = h.solve(dev(f), tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(host(x) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])
    rng = np.random.default_rng(256)
    for l in (0, 1):
        Al, Pl = ho.matrix(l, "A"), ho.matrix(l, "P")
        m = ho.smoother(l)
        fl = rng.standard_normal(Al.nrows)
        xl = rng.standard_normal(Al.nrows)
        e = rng.standard_normal(Pl.ncols)
        mf = m * fl
        y = torch.empty(Al.nrows, dtype=torch.float64, device="cuda")
        h.level_op_ex(l, amgb.OP_RES0_MF, in0=dev(fl), in1=dev(mf), out0=y)
        check_rows(host(y), fl - oracle.spmv(Al, mf), row_bound(Al, mf, fl), f"l{l} res0")
        h.level_op_ex(l, amgb.OP_PROL0_MF, in0=dev(e), in1=dev(mf), out0=y)
        check_rows(host(y), mf + oracle.spmv(Pl, e), row_bound(Pl, e, mf), f"l{l} prolong0")
        rho = h.level_op_ex(l, amgb.OP_RELAX_RHO, in0=dev(xl), in1=dev(fl), out0=y)
        ref = ho.relax(l, fl, xl)
        b = np.abs(m) * row_bound(Al, xl, fl) + 4 * U * (np.abs(xl) + np.abs(m * (fl - oracle.spmv(Al, xl))))
        check_rows(host(y), ref, b, f"l{l} relax+rho")
        assert abs(rho - np.dot(fl, ref)) <= dot_bound(fl, ref, 0.0, b)
