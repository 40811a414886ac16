"""Mixed-precision V-cycle (params.precision = 1): the
V-cycle reads fp32 copies of the hierarchy values; vectors, arithmetic and the
Krylov method stay fp64.  Its own parity bar:
* V-cycle: |z_mixed - z_fp64| <= 1e-5 |z_fp64| (fp32 rounding of the values,
  u_32 = 6e-8, amplified through the smoothers and the coarse solve);
* solve: converges to the same tolerance (true residual <= tol), iterations
  within +-1 of the fp64 oracle, |x - x_oracle| <= 1e-6 |x_oracle| (both satisfy
  |f - A x| <= 1e-8 |f|).  GPU only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


CASES = [("poisson", 32, {}), ("poisson_perm", 24, {}), ("varcoef", 24, {"relax": "chebyshev"}),
         ("convdiff", 20, {"relax": "damped_jacobi", "solver": "bicgstab"}), ("poisson", 20, {"npre": 2})]


@pytest.mark.parametrize("gen,n,kw", CASES)
def test_mixed_precision_solve(gen, n, kw):
    p, c, v, f = synth.problem(gen, n)
    kw = dict(kw, coarse_enough=100)
    hm = amgb.setup(p, c, v, precision="mixed", **kw)
    hd = amgb.setup(p, c, v, **kw)
    r = synth.random_vector(len(f))
    zm = hm.precond(dev(r)).cpu().numpy()
    zd = hd.precond(dev(r)).cpu().numpy()
    assert np.linalg.norm(zm - zd) <= 1e-5 * np.linalg.norm(zd)
    assert np.linalg.norm(zm - zd) > 0  # the fp32 values are really used
    x, it, rel, st = hm.solve(dev(f), tol=1e-8, maxiter=200)
    assert st == amgb.OK and rel <= 1.01e-8
    A = oracle.Csr(p, c, v)
    okw = {k: val for k, val in kw.items() if k != "solver"}
    fn = oracle.bicgstab if kw.get("solver") == "bicgstab" else oracle.cg
    o = fn(A, f, tol=1e-8, maxiter=200, hier=oracle.Hierarchy(A, **okw))
    assert abs(it - o["iters"]) <= 1, (it, o["iters"])
    xh = x.cpu().numpy()
    assert np.linalg.norm(xh - o["x"]) <= 1e-6 * np.linalg.norm(o["x"])
    # fewer algorithmic bytes per V-cycle than fp64
    assert hm.level_info(0)["alg_bytes_vcycle"] < hd.level_info(0)["alg_bytes_vcycle"]
