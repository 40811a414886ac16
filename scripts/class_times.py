"""In-graph time per kernel class (CUDA-event record nodes around each launch of one
class at a time, amg_set_profile) against the unprofiled solve time: where the solve
time goes, and how much is launch gaps / tails between kernels."""
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
ap.add_argument("--solves", type=int, default=5)
a = ap.parse_args()
p, c, v, f = synth.problem(a.problem, a.n)
h = amgb.setup(p, c, v, {})
fd = torch.from_numpy(f).cuda()
x = torch.zeros_like(fd)
s = torch.cuda.Stream()


def run(mask):
    h.set_profile(mask)
    with torch.cuda.stream(s):
        for _ in range(2):
            x.zero_()
            h.solve(fd, x, tol=1e-8, maxiter=200)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = [0.0] * len(amgb.PROF_CLASSES)
        gb = [0.0] * len(amgb.PROF_CLASSES)
        nl = [0] * len(amgb.PROF_CLASSES)
        e0.record(s)
        for _ in range(a.solves):
            x.zero_()
            _, it, rel, st = h.solve(fd, x, tol=1e-8, maxiter=200)
            st_ = h.stats()
            for c_ in range(len(ms)):
                ms[c_] += st_["prof_ms"][c_]
                gb[c_] += st_["prof_bytes"][c_] / 1e9
                nl[c_] += st_["prof_launches"][c_]
        e1.record(s)
        torch.cuda.synchronize()
    h.set_profile(0)
    return e0.elapsed_time(e1) / a.solves, [m / a.solves for m in ms], [g / a.solves for g in gb], \
        [n // a.solves for n in nl], it


base, _, _, _, it = run(0)
print(f"unprofiled solve: {base:.3f} ms ({it} iterations)")
tot = 0.0
for c_, name in enumerate(amgb.PROF_CLASSES):
    t, ms, gb, nl, _ = run(1 << c_)
    tot += ms[c_]
    bw = gb[c_] / (ms[c_] / 1e3) if ms[c_] > 0 else 0.0
    print(f"class {name:14s}: {ms[c_]:8.3f} ms/solve  {nl[c_]:5d} launches  {gb[c_]:7.2f} GB  {bw:7.0f} GB/s"
          f"  (solve with these events: {t:.3f} ms)")
print(f"sum of classes {tot:.3f} ms vs unprofiled {base:.3f} ms: gaps/tails {base - tot:.3f} ms")
