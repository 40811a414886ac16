"""Execution-policy choices that must not change results: the
opt-in fused CG iteration (AMGB_CG_FUSION=1) computes the same fma sequence
as the plain unfused iteration, so x is bitwise equal either way.  The unfused
iteration's update kernel also writes m o r for the level-0 residual (mf0); its
prolongation then adds (m o f) + P e instead of fma(m, f, P e): one rounding
apart, so equal iteration counts and x within 1e-12.  GPU only."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def solve_with(env, gen, n):
    p, c, v, f = synth.problem(gen, n)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        h = amgb.setup(p, c, v, coarse_enough=200)
        x, it, rel, st = h.solve(dev(f), tol=1e-8)
        torch.cuda.synchronize()
        return x.cpu().numpy(), it, rel, h.stats()["flags"]
    finally:
        for k, val in old.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val


@pytest.mark.parametrize("gen,n,fused_by_default", [("poisson", 40, 0), ("poisson_perm", 40, 0)])
def test_fusion_policy_and_bitwise_equal(gen, n, fused_by_default):
    x0, it0, rel0, fl0 = solve_with({}, gen, n)
    assert fl0 & 1 == fused_by_default
    x1, it1, rel1, fl1 = solve_with({"AMGB_CG_FUSION": "1"}, gen, n)
    x2, it2, rel2, fl2 = solve_with({"AMGB_CG_FUSION": "0", "AMGB_NO_MF0": "1"}, gen, n)
    x3, it3, rel3, fl3 = solve_with({"AMGB_CG_FUSION": "0"}, gen, n)
    assert fl1 & 1 == 1 and fl2 & 1 == 0 and fl3 & 1 == 0
    assert it0 == it1 == it2 == it3 and rel1 == rel2
    assert np.array_equal(x1, x2)
    assert np.array_equal(x0, x1 if fused_by_default else x3)
    assert np.linalg.norm(x3 - x2) <= 1e-12 * np.linalg.norm(x2)
