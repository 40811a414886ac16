"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel
shares of the step and per-position times within one Krylov iteration."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    names = [re.sub(r"amgb::", "", r[ki]) for r in data]
    t = [float(r[vi].replace(",", "")) for r in data]  # ns
    return names, t


def short(n):
    m = re.match(r"void (\w+)<(.*?)>\(", n)
    return (m.group(1) + "<" + m.group(2)[:48] + ">") if m else n.split("(")[0][:60]


def main(path, marker="VCgUpdate"):
    names, t = load(path)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v in zip(names, t):
        tot[short(n)] += v
        cnt[short(n)] += 1
    # setup-phase kernels (GPU setup k_*, format conversion cv_*, CUB, torch) are
    # listed apart: the shares are of the solve kernels
    setup = {k for k in tot if re.match(r"(<unnamed>::)?(k_|cv_)|cub::|void cub|at::|void at::", k)}
    T = sum(v for k, v in tot.items() if k not in setup)
    S = sum(tot[k] for k in setup)
    print(f"# {len(t)} launches; solve kernels {T / 1e6:.3f} ms, setup/other kernels {S / 1e6:.3f} ms "
          "(ncu: serialised, cold-cache)")
    print("# share of solve  total_ms  launches  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        if k not in setup:
            print(f"{100 * v / T:6.2f}% {v / 1e6:9.3f} {cnt[k]:6d}  {k}")
    print("# setup / other kernels")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        if k in setup:
            print(f"   --  {v / 1e6:9.3f} {cnt[k]:6d}  {k}")
    idx = [i for i, n in enumerate(names) if marker in n]
    if len(idx) > 2:
        per = collections.Counter(b - a for a, b in zip(idx, idx[1:])).most_common(1)[0][0]
        seqs = [(a + 1, b + 1) for a, b in zip(idx, idx[1:]) if b - a == per]
        print(f"\n# one Krylov iteration = {per} launches; mean over {len(seqs)} iterations (us)")
        it_tot = 0.0
        for k in range(per):
            vals = [t[a + k] for a, _ in seqs]
            m = sum(vals) / len(vals) / 1e3
            it_tot += m
            print(f"{k:3d} {m:9.1f}  {short(names[seqs[0][0] + k])}")
        print(f"# iteration total {it_tot:.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
