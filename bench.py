#!/usr/bin/env python
"""bench.py -- AMG-preconditioned CG solve phase on B200 (arXiv 1811.05704).

Headline (BASELINE.json metric): solve time and V-cycles/s of CG + smoothed-
aggregation AMG (SPAI-0) on the 3D Poisson problem 256^3 (16,777,216 unknowns,
117,047,296 nonzeros; Eq. (2)), tolerance 1e-8, with the
HBM-roofline fraction of the dominant kernel class.

One "step" = one full solve from x = 0 to rel. residual 1e-8 (all of §8(a):
V-cycle kernels, Krylov updates, dots, convergence tests), inputs resident in
HBM.  value = V-cycles per second over the K timed steps (whole job).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl amgb|reference]
                  [--problem poisson|poisson_perm|varcoef|convdiff] [--n 256]

--impl reference times the oracle (plain fp64 C, oracle/) on the host cores:
one step = one full oracle solve of the same system (V-cycles / time, as
cpu_baseline).

Multi-GPU (torchrun, N > 1): strong scaling -- the same global system is
row-partitioned over the N GPUs (halo exchange, all-reduce and coarse-level
all-gather over NCCL); time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
METRIC = "AMG-CG V-cycles/s, 3D Poisson 256^3 (solve time in config.solve_ms)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="amgb", choices=["amgb", "reference"])
    ap.add_argument("--problem", default="poisson")
    ap.add_argument("--n", "--size", dest="n", type=int, default=256)
    ap.add_argument("--relax", default=None)
    ap.add_argument("--solver", default=None)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--maxiter", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--batch", type=int, default=1,
                    help="k > 1: k right-hand sides per solve (amg_solve_batched); value counts column V-cycles")
    ap.add_argument("--precision", default="double", choices=["double", "mixed"],
                    help="mixed: fp32 hierarchy values in the V-cycle (not the headline; SURVEY §8f rank 2)")
    ap.add_argument("--reorder", default="auto", choices=["auto", "on", "off"],
                    help="locality reordering of the device store (params reorder 2 / 1 / 0)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="weak: BASELINE configs[4], Poisson on 256 x 256 x 256N (one 256^3 block per GPU); "
                         "value = unknown-V-cycles/s (rows x V-cycles / s)")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


PROBLEM_DEFAULTS = {  # BASELINE.json configs -> solver settings
    "poisson": dict(relax="spai0", solver="cg", maxiter=100),
    "poisson_perm": dict(relax="spai0", solver="cg", maxiter=100),
    "varcoef": dict(relax="chebyshev", solver="cg", maxiter=200),
    "convdiff": dict(relax="damped_jacobi", solver="bicgstab", maxiter=200),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def problem_arrays(name, n):
    ptr, col, val, f = synth.problem(name, n)
    return ptr, col, val, f


def workload_name(args, cfg):
    w = f"{args.problem}{args.n}^3_{cfg['solver']}_sa_{cfg['relax']}"
    return w + ("_mixed" if getattr(args, "precision", "double") == "mixed" else "")


def oracle_solver(cfg):
    import oracle
    return {"cg": oracle.cg, "bicgstab": oracle.bicgstab, "gmres": oracle.gmres, "idrs": oracle.idrs}[cfg["solver"]]


def cpu_baseline_full_solve(ptr, col, val, f, cfg, tol, maxiter):
    """The oracle as it stands on the host cores: untimed setup, then one full
    solve of the same system (timed).  Also returns its iterations/solution for
    the full-size parity check."""
    import oracle
    A = oracle.Csr(ptr, col, val)
    t0 = time.perf_counter()
    hier = oracle.Hierarchy(A, relax=cfg["relax"])
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = oracle_solver(cfg)(A, f, tol=tol, maxiter=maxiter, hier=hier)
    t_solve = time.perf_counter() - t0
    vcyc = res.get("vcycles", res["iters"])
    # a bounded 1-thread sample: one oracle V-cycle (or_precond)
    # on the same hierarchy with the OpenMP row loops on one thread
    one = None
    try:
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        gomp.omp_get_max_threads.restype = ctypes.c_int
        nt = gomp.omp_get_max_threads()
        gomp.omp_set_num_threads(1)
        try:
            r = synth.random_vector(len(f))
            t0 = time.perf_counter()
            hier.precond(r)
            one = time.perf_counter() - t0
        finally:
            gomp.omp_set_num_threads(nt)
    except OSError:
        pass
    return dict(setup_s=t_setup, solve_s=t_solve, iters=res["iters"], vcycles=vcyc, x=res["x"],
                rel=res["rel_resid"], one_thread_vcycle_s=one)


def cpu_info():
    """Host CPU model name and core count (the oracle baseline's machine)."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_threads():
    """Threads the oracle's OpenMP row loops use (OMP_NUM_THREADS, else all cores)."""
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v and v.isdigit() else os.cpu_count()


def run_reference(args, cfg):
    """--impl reference: the oracle timed on the host cores (rank 0 only).  One
    step = one full oracle solve of the same system from x = 0 to the same
    tolerance (setup untimed), value = V-cycles / time, exactly as cpu_baseline."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # rank 0 alone runs the oracle: give it the host cores (torchrun exports
    # OMP_NUM_THREADS=1 to every rank; libgomp reads it when the oracle loads)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import oracle
    ptr, col, val, f = problem_arrays(args.problem, args.n)
    A = oracle.Csr(ptr, col, val)
    t0 = time.perf_counter()
    hier = oracle.Hierarchy(A, relax=cfg["relax"])
    t_setup = time.perf_counter() - t0
    fn = oracle_solver(cfg)
    for _ in range(args.warmup):
        fn(A, f, tol=args.tol, maxiter=cfg["maxiter"], hier=hier)
    vc, iters = 0, 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = fn(A, f, tol=args.tol, maxiter=cfg["maxiter"], hier=hier)
        vc += r.get("vcycles", r["iters"])
        iters = r["iters"]
    dt = time.perf_counter() - t0
    cores = oracle_threads()
    value = vc / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "V-cycles/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth/)",
        "config": {"workload": workload_name(args, cfg),
                   "step": f"one full oracle solve from x = 0 to tol {args.tol} ({iters} iterations)",
                   "oracle_setup_s": t_setup, **cpu_info()},
        "cpu_baseline": {"value": value, "unit": "V-cycles/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} full oracle solves of the {args.n}^3 system "
                                   f"({iters} iterations each; setup untimed)"},
        "e2e": {"value": value, "unit": "V-cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_batched(args, cfg, h, f, n, nnz, infos, setup_s, local, stream):
    """k right-hand sides per solve through amg_solve_batched (1 GPU)."""
    import torch
    k = args.batch
    rng = np.random.default_rng(synth.SEED_VEC)
    F = rng.standard_normal((k, n))
    F[0] = f
    Fd = torch.from_numpy(F).cuda()
    X = torch.zeros_like(Fd)
    tol, maxiter = args.tol, cfg["maxiter"]
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            X.zero_()
            h.solve_batched(Fd, X, tol=tol, maxiter=maxiter)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cols, alg, launches = 0, 0.0, 0
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for _ in range(args.steps):
                X.zero_()
                _, its, rels, st = h.solve_batched(Fd, X, tol=tol, maxiter=maxiter)
                s = h.stats()
                cols += int(np.sum(its))
                alg += s["alg_bytes"]
                launches += s["kernel_launches"]
            ev1.record(stream)
            torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    peak, peak_src = peaks()
    line = {
        "metric": METRIC + " [batched: column V-cycles/s]", "value": cols / (ms / 1e3), "unit": "column V-cycles/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: f = 1 and k-1 seeded N(0,1) right-hand sides",
        "config": {"workload": workload_name(args, cfg) + f"_batch{k}", "n": n, "nnz": nnz, "batch": k,
                   "iters_per_column": [int(v) for v in its], "rel_resid_max": float(np.max(rels)),
                   "solve_alg_GBps": alg / (ms / 1e3) / 1e9, "solve_roofline_frac": alg / (ms / 1e3) / 1e9 / peak,
                   "levels": len(infos), "setup_s": setup_s},
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = dict(PROBLEM_DEFAULTS[args.problem])
    if args.relax:
        cfg["relax"] = args.relax
    if args.solver:
        cfg["solver"] = args.solver
    if args.maxiter:
        cfg["maxiter"] = args.maxiter
    if args.impl == "reference":
        return run_reference(args, cfg)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # host setup threads: share the host cores between the ranks of this node
    # (multi-GPU: rank 0 alone builds and partitions the hierarchy -- the scattered
    # setup -- so it gets the cores; torchrun exports OMP_NUM_THREADS=1 to every rank)
    if world > 1 and int(os.environ.get("RANK", "0")) == 0:
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    else:
        os.environ.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // world)))

    import torch
    import torch.distributed as dist

    import paper_1811_05704_b200 as amgb

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TEST ONLY (AMGB_BENCH_ONE_GPU=1): every rank on GPU 0, torch.distributed over
    # gloo and the library's host shared-memory transport (AMGB_TRANSPORT=shm), so
    # this N > 1 path runs end to end on a one-GPU box; numbers from it are not
    # multi-GPU measurements
    one_gpu = world > 1 and os.environ.get("AMGB_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
        os.environ["AMGB_TRANSPORT"] = "shm"
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    weak = args.scaling == "weak"
    if weak and args.problem != "poisson":
        raise SystemExit("--scaling weak is the Poisson configuration (BASELINE.json configs[4])")
    # multi-GPU: scattered setup -- rank 0 alone builds the global matrix and
    # the hierarchy; the other ranks only need their slice of f
    if rank == 0 or world == 1:
        ptr, col, val, f = synth.weak_poisson(world, args.n) if weak else problem_arrays(args.problem, args.n)
        n, nnz = len(f), int(ptr[-1])
    else:
        ptr = col = val = f = None
        n = args.n ** 3 * world if weak else synth.problem_rows(args.problem, args.n)
        nnz = None
    prm = {"precond.relax.type": cfg["relax"], "solver.type": cfg["solver"], "precision": args.precision}
    torch.empty(1, device=f"cuda:{local}")  # CUDA context creation stays outside setup_s
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world == 1:
        h = amgb.setup(ptr, col, val, prm, device=local, use_graph=0 if args.no_graph else 1,
                       reorder={"auto": 2, "on": 1, "off": 0}[args.reorder])
        r0, r1 = 0, n
    else:
        # strong scaling: the global system row-partitioned over the ranks, halo
        # exchange / all-reduce / coarse all-gather over NCCL
        uid = torch.zeros(128, dtype=torch.uint8, device="cpu" if one_gpu else "cuda")
        if rank == 0:
            uid.copy_(torch.tensor(list(amgb.nccl_unique_id() if not one_gpu else os.urandom(128)),
                                   dtype=torch.uint8))
        dist.broadcast(uid, 0)
        h = amgb.setup_dist(ptr, col, val, nranks=world, rank=rank, nccl_id=bytes(uid.cpu().tolist()),
                            params=prm, device=local, use_graph=0 if args.no_graph else 1, n=n)
        st = h.dist_info()["row_starts"]
        r0, r1 = int(st[rank]), int(st[rank + 1])
        if f is None:
            f = np.empty(n)
            f[r0:r1] = np.ones(r1 - r0) if weak else synth.rhs_slice(args.problem, args.n, r0, r1)
    setup_s = time.perf_counter() - t0
    infos = [h.level_info(l) for l in range(h.nlevels)]
    nl = r1 - r0

    stream = torch.cuda.Stream()
    fd = torch.from_numpy(np.ascontiguousarray(f[r0:r1])).cuda()
    x = torch.zeros_like(fd)
    tol, maxiter = args.tol, cfg["maxiter"]
    if args.batch > 1:
        return run_batched(args, cfg, h, f, n, nnz, infos, setup_s, local, stream)

    def timed_solves(profile_mask):
        """K timed solves from x = 0 (barrier + synchronize on both sides, CUDA
        events on the solve stream)."""
        h.set_profile(profile_mask)
        x.zero_()
        h.solve(fd, x, tol=tol, maxiter=maxiter)  # (re)build the graph for this mode
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        acc = dict(iters=[], vc=0, launches=0, prof_ms=0.0, prof_bytes=0.0, prof_launch=0, alg_bytes=0.0,
                   status=[], rel=[])
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for _ in range(args.steps):
                x.zero_()
                _, it, rel, st = h.solve(fd, x, tol=tol, maxiter=maxiter)
                s = h.stats()
                acc["iters"].append(it)
                acc["vc"] += s["vcycles"]
                acc["launches"] += s["kernel_launches"]
                acc["prof_ms"] += s["prof_ms"][0]
                acc["prof_bytes"] += s["prof_bytes"][0]
                acc["prof_launch"] += s["prof_launches"][0]
                acc["alg_bytes"] += s["alg_bytes"]
                acc["status"].append(st)
                acc["rel"].append(rel)
                acc["flags"] = s["flags"]
            ev1.record(stream)
            torch.cuda.synchronize()
        acc["ms"] = ev0.elapsed_time(ev1)
        acc["clocks"] = clk.summary()
        barrier()
        h.set_profile(0)
        return acc

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            x.zero_()
            h.solve(fd, x, tol=tol, maxiter=maxiter)
        # (A) headline: production path (device-side Krylov loop in one CUDA graph)
        A = timed_solves(0)
        # (B) roofline: the same solves with CUDA-event nodes around the dominant
        #     kernel class (level-0 A passes) inside the iteration graph
        B = timed_solves(1 << 0)
    elapsed_ms = A["ms"]
    iters_all, vc_total, launches, alg_bytes, statuses, rels = (A["iters"], A["vc"], A["launches"],
                                                                 A["alg_bytes"], A["status"], A["rel"])
    prof_ms, prof_bytes, prof_launch = B["prof_ms"], B["prof_bytes"], B["prof_launch"]
    clk_summary = A["clocks"]
    tdev = "cpu" if one_gpu else "cuda"  # gloo (test only) reduces host tensors
    t_local = torch.tensor([elapsed_ms], dtype=torch.float64, device=tdev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_max_ms = float(t_local.item())
    # one global solve per step: the job's V-cycles are those of the solve
    value = float(vc_total) / (t_max_ms / 1e3)
    if weak:  # whole-job work of a weak-scaling step: rows x V-cycles
        value *= n

    # ---- end-to-end through the public API with HOST buffers (amg_solve_host_stream)
    e2e = None
    if not args.no_e2e:
        # pinned host f (input) and x (solution); zero initial guess (x0 = NULL)
        fh = torch.from_numpy(np.ascontiguousarray(f[r0:r1])).pin_memory().numpy()
        xh = torch.zeros(nl, dtype=torch.float64).pin_memory().numpy()
        # amg_solve_host_stream: one system per step, each step copies its f in
        # and its x out; the copies overlap the neighbouring steps' solves
        with torch.cuda.stream(stream):
            w = max(2, args.warmup // 2)
            h.solve_host_stream([fh] * w, [xh] * w, tol=tol, maxiter=maxiter)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, _, _, vcs, _ = h.solve_host_stream([fh] * args.steps, [xh] * args.steps, tol=tol, maxiter=maxiter)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            vc_e = sum(vcs)
        te = torch.tensor([dt], dtype=torch.float64, device=tdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(vc_e) / float(te.item()) * (n if weak else 1),
               "unit": "unknown-V-cycles/s" if weak else "V-cycles/s",
               "h2d_bytes_per_step": 8 * nl, "d2h_bytes_per_step": 8 * nl,
               "ms_per_step": 1e3 * float(te.item()) / args.steps,
               "timing": "host wall clock around one amg_solve_host_stream call of K systems (per system: "
                         "H2D f + solve + D2H x from/to pinned host buffers, zero initial guess; the copies of "
                         "system j+1's f and system j-1's x overlap system j's solve), max over ranks"}

    peak, peak_src = peaks()
    achieved = (prof_bytes / (prof_ms / 1e3)) / 1e9 if prof_ms > 0 else None
    solve_gbs = (alg_bytes / (elapsed_ms / 1e3)) / 1e9
    # roofline.traffic: DRAM bytes per level-0 A-pass launch from the committed
    # ncu --set full capture (profiles/ncu_traffic.json); ncu cannot run inside
    # this process, so the capture names the libamgb.so it profiled and the line
    # says whether that is the build running here
    traffic, traffic_src = None, None
    try:
        import hashlib
        with open(amgb.LIB_PATH, "rb") as fh_:
            lib_sha = hashlib.sha256(fh_.read()).hexdigest()
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh_:
            tj = json.load(fh_)
        if tj.get("workload") == workload_name(args, cfg):
            traffic = tj.get("a0_pass_bytes_per_launch")
            traffic_src = {"file": "profiles/ncu_traffic.json", "capture": tj.get("source"),
                           "lib_sha256": tj.get("lib_sha256"), "this_lib_sha256": lib_sha,
                           "same_build": tj.get("lib_sha256") == lib_sha}
    except Exception:
        pass

    # ---- CPU baseline: the oracle on this host (rank 0, N = 1 only)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not weak:
        cb = cpu_baseline_full_solve(ptr, col, val, f, cfg, tol, maxiter)
        cpu = {"value": cb["vcycles"] / cb["solve_s"], "unit": "V-cycles/s", "cores": oracle_threads(),
               "kind": "oracle",
               "sample": f"one full oracle solve of the same {args.n}^3 system ({cb['iters']} iterations, "
                         f"{cb['solve_s']:.1f} s; oracle setup {cb['setup_s']:.1f} s untimed)",
               **cpu_info(),
               "one_thread": None if cb["one_thread_vcycle_s"] is None else {
                   "value": 1.0 / cb["one_thread_vcycle_s"], "unit": "V-cycles/s (V-cycle only)", "cores": 1,
                   "sample": "one oracle V-cycle (or_precond) of the same hierarchy, OpenMP on 1 thread"}}
        xg = x.cpu().numpy()  # N = 1: the full solution
        parity = {"oracle_iters": cb["iters"], "gpu_iters": iters_all[-1],
                  "x_rel_diff": float(np.linalg.norm(xg - cb["x"]) / np.linalg.norm(cb["x"])),
                  "oracle_rel_resid": cb["rel"]}

    if rank == 0:
        line = {
            "metric": METRIC if not weak else
            "AMG-CG unknown-V-cycles/s, 3D Poisson weak scaling 256^3 per GPU (BASELINE configs[4])",
            "value": value, "unit": "unknown-V-cycles/s" if weak else "V-cycles/s", "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64" if args.precision == "double" else "f64 (V-cycle matrix values f32)",
            "data": "synthetic (seeded generators, synth/): 7-point FD Poisson, f = 1",
            "config": {
                "workload": (f"poisson{args.n}x{args.n}x{args.n * world}_weak_cg_sa_spai0" if weak
                             else workload_name(args, cfg)), "n": n, "nnz": nnz, "tol": tol,
                "solver": cfg["solver"], "relax": cfg["relax"], "coarsening": "smoothed_aggregation",
                "parallelism": "1 GPU" if world == 1 else
                f"row partition over {world} GPUs (NCCL halo exchange + all-reduce; levels < "
                f"{h.dist_info()['first_replicated']} distributed, coarser replicated)",
                "levels": len(infos), "rows_per_level": [i["rows"] for i in infos],
                "nnz_per_level": [i["nnz_A"] for i in infos],
                "reordered_store": bool(A.get("flags", 0) & 2),
                "dict_slice_frac_A0": round(infos[0]["dict_slices_A"] / max(1, (h.vec_len + 31) // 32), 4),
                "iters_per_solve": iters_all[-1], "rel_resid": rels[-1], "status": statuses[-1],
                "solve_ms": t_max_ms / args.steps, "setup_s": setup_s,
                "setup": "hierarchy built on the GPU (strength, aggregation, P, R, RAP, smoother; the coarsest "
                         "dense inverse on the host), device formats + value indexing; CUDA context created "
                         "before the timer",
                "l2": "inputs larger than L2 (level-0 matrix %.2f GB + hierarchy vs 126 MB L2); no flush"
                      % (12e-9 * infos[0]["nnz_A"]),
                "solve_alg_GBps": solve_gbs, "solve_roofline_frac": solve_gbs / peak,
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "kernel": "level-0 A-pass kernels (one kernel template on A0 in the format pick_format chose: sell_tma at 256^3; res0 / relax+rho / cg-dir+sigma / initial and true residual)",
                "store": "A0 %s values, %s column indices (bytes_per_launch counts what this store moves)" % (
                    {0: "fp64", 1: "8-bit indexed", 2: "16-bit indexed"}[infos[0].get("vidx_A", 0)],
                    "offset-dictionary" if infos[0]["dict_slices_A"] else "explicit"),
                "launches_timed": prof_launch, "bytes_per_launch": prof_bytes / max(prof_launch, 1),
                "ms_per_launch": prof_ms / max(prof_launch, 1), "peak_source": peak_src,
                "timed_in": "a second timed region of the same K solves with CUDA-event record nodes "
                            "around each level-0 A pass inside the iteration graph "
                            f"(that region: {B['ms'] / args.steps:.2f} ms per solve)",
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk_summary,
            "parity_full_size": parity,
        }
        out = json.dumps(line)
        print(out, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh_:
                fh_.write(out + "\n")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
