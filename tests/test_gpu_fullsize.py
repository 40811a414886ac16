"""BASELINE.json configurations at FULL size against the oracle (GPU only).

* configs[2] (256^3 variable-coefficient Poisson, Chebyshev smoother): one
  preconditioner application z = M r on the full hierarchy, element by element
  against the oracle's V-cycle (1e-12 relative), and the converged solve checked
  through its true residual computed by the oracle's SpMV.
* configs[3] (200^3 convection-diffusion, BiCGStab + damped Jacobi): the whole
  solve against the oracle's (iterations +-1; x within 1e-8 at equal count).
(configs[0] and configs[1] at full size: tests/test_gpu_parity.py; the headline
256^3 Poisson solve is checked against a full oracle solve by bench.py's
parity_full_size on every bench run.)"""
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
