"""Interleaved in-process A/B of execution variants on one system (GPU).

Variants are (setup env, solve env) pairs; each round runs every variant once
(one untimed solve after a switch, then --solves timed solves, CUDA events on the
handle's stream), rounds repeat so clock/power drift hits all variants alike.
Prints the median ms per solve per variant and the iteration counts.

  python scripts/ab_inproc.py --n 256 --variants "base:;nodict:AMGB_NO_DICT=1|;unfused:|AMGB_CG_FUSION=0"
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def parse_env(s):
    out = {}
    for kv in filter(None, s.split(",")):
        k, v = kv.split("=", 1)
        out[k] = v
    return out


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="poisson")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--variants", required=True, help="name:setup_env|solve_env[|setup kwargs k=v,...];...")
    a = ap.parse_args()
    p, c, v, f = synth.problem(a.problem, a.n)
    fd = torch.from_numpy(f).cuda()
    variants = []
    handles = {}
    for spec in a.variants.split(";"):
        name, envs = spec.split(":", 1)
        fields = envs.split("|") + ["", ""]
        se, so, kw = parse_env(fields[0]), parse_env(fields[1]), parse_env(fields[2])
        key = (tuple(sorted(se.items())), tuple(sorted(kw.items())))
        if key not in handles:
            handles[key] = with_env(se, lambda: amgb.setup(p, c, v, **kw))
        variants.append((name, handles[key], so))
    times = {n: [] for n, _, _ in variants}
    iters = {}
    x = torch.zeros_like(fd)
    for r in range(a.rounds):
        for name, h, so in variants:
            def run():
                x.zero_()
                h.solve(fd, x=x, tol=1e-8)  # untimed: graph (re)capture after a switch
                torch.cuda.synchronize()
                ms = []
                for _ in range(a.solves):
                    x.zero_()
                    _, it, rel, st = h.solve(fd, x=x, tol=1e-8)
                    ms.append(h.stats()["solve_ms"])
                    iters[name] = (it, h.stats()["flags"])
                return ms
            times[name] += with_env(so, run)
    for name, _, _ in variants:
        t = times[name]
        print(f"{name:12s} median {statistics.median(t):8.3f} ms  min {min(t):8.3f}  max {max(t):8.3f}  "
              f"iters/flags {iters[name]}")


if __name__ == "__main__":
    main()
