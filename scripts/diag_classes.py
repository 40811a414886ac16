"""Per-kernel-class device time of a 256^3 solve (event nodes around every
launch, host-loop graph) vs the solve time: how much is launch gaps / idle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p, c, v, f = synth.poisson3d(n)
h = amgb.setup(p, c, v)
fd = torch.from_numpy(f).cuda()
for mask in (0, 0xFF):
    h.set_profile(mask)
    for _ in range(3):
        x, it, rel, st = h.solve(fd)
    tot = {k: 0.0 for k in amgb.PROF_CLASSES}
    solve = 0.0
    for _ in range(5):
        x, it, rel, st = h.solve(fd)
        s = h.stats()
        solve += s["solve_ms"]
        for k, ms in zip(amgb.PROF_CLASSES, s["prof_ms"]):
            tot[k] += ms
    print(f"mask {mask:#x}: solve {solve / 5:.2f} ms, iters {it}, classes (ms/solve):",
          {k: round(t / 5, 3) for k, t in tot.items()}, "sum", round(sum(tot.values()) / 5, 2), flush=True)
