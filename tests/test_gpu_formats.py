"""Per-row oracle parity of every fused kernel of the solve phase, in every
device format the headline runs (VERDICT r1 "next #1").  GPU only (-m gpu).

pick_format (amgb.cu) stores a matrix with >= 65,536 rows as TMA-staged SELL-32
(narrow, unpadded rows: A0 at 256^3), TMA-staged CSR (narrow rows that SELL-32
would pad by > 15 %: P0, P1; padded wide restrictions: R0, R1) or SELL-32 (the
wide coarse A: A1, A2), and smaller
ones as row-block CSR; AMGB_FORMAT = sell | tma | tmacsr forces a format on
every level, AMGB_NO_DICT=1 stores the TMA format with explicit column indices
instead of the per-slice offset dictionary.  Each case runs every op of Algorithm 2
 and of the CG iteration
through amg_level_op / amg_level_op_ex -- the op structs and kernel templates the
solve launches -- and compares every output row with the oracle on the same
seeded inputs under the a-priori rounding bound of a reordered / FMA row sum:

    |y_i - y_oracle_i| <= 8 (len_i + 2) u (|M| |v| + |g|)_i,   u = 2^-53,

where v is the gathered vector and g the row-local term of the epilogue; fused
dot products are bounded by (n + 2) u sum|a_i b_i| plus the propagated row
bounds.  Outputs that are one IEEE operation of GPU values (m o f written by the
restriction and the CG update) must be bitwise equal.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402

U = 2.0 ** -53


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def empty(n):
    return torch.empty(n, dtype=torch.float64, device="cuda")


def lens(M):
    return np.diff(M.ptr).astype(float)


def absdot(M, v):
    return oracle.spmv(oracle.Csr(M.ptr, M.col, np.abs(M.val), M.ncols), np.abs(v))


def row_bound(M, v, g=0.0):
    """8 (len + 2) u (|M||v| + |g|) per row."""
    return 8 * (lens(M) + 2) * U * (absdot(M, v) + np.abs(g)) + 1e-300


def check_rows(y, ref, bound, what):
    err = np.abs(y - ref)
    bad = np.flatnonzero(err > bound)
    assert bad.size == 0, f"{what}: {bad.size} rows over the bound, first {bad[:5]}, max err {err.max():.3e}"


def dot_bound(a, b, da=0.0, db=0.0):
    """|(a, b)_gpu - (a_ref, b_ref)| for a reordered sum of n products plus the
    propagated row errors da, db of the operands."""
    n = len(a)
    return (n + 2) * U * np.sum(np.abs(a * b)) + np.sum(np.abs(da) * np.abs(b)) + np.sum(np.abs(a) * np.abs(db)) \
        + 1e-300


def okw(kw):
    o = dict(kw)
    if "coarsening" in o:
        o["smoothed"] = 1 - o.pop("coarsening")
    return o


# (generator, n, setup keywords): >= 65,536 rows on level 0 so `auto` stores A0 and
# P0 in the TMA format and R0 in SELL; 41^3 is ragged (68,921 rows: not a
# multiple of the 32-row slice or the 256-row tile)
CASES = [
    ("poisson", 41, {}),
    ("poisson_perm", 42, {"reorder": 0}),           # unstructured order, explicit indices
    ("poisson_perm", 41, {}),                       # same, reordered store (RCM)
    ("varcoef", 41, {"relax": "chebyshev"}),
    ("convdiff", 41, {"relax": "damped_jacobi"}),
]
FORMATS = {  # env of the device store
    "auto": {},
    "sell": {"AMGB_FORMAT": "sell"},
    "tma": {"AMGB_FORMAT": "tma"},
    "tma_explicit": {"AMGB_FORMAT": "tma", "AMGB_NO_DICT": "1"},
    "tmacsr": {"AMGB_FORMAT": "tmacsr"},
}


def sell_padding(M):
    """Stored / nnz of M as SELL-32 (every row at its 32-row slice's longest)."""
    ln = lens(M)
    pad = np.zeros(-(-len(ln) // 32) * 32)
    pad[:len(ln)] = ln
    return 32 * pad.reshape(-1, 32).max(axis=1).sum() / max(M.nnz, 1) if M.nrows else 1.0


def expected_fmt(fmt, M, role="A"):
    if fmt == "sell":
        return amgb.FMT_SELL
    if fmt == "tmacsr":
        return amgb.FMT_SELL if tcsr_wide(M) else amgb.FMT_TMACSR
    if fmt.startswith("tma"):
        return amgb.FMT_SELL if tma_wide(M) else amgb.FMT_TMA
    if M.nrows < 65536:
        return amgb.FMT_CSR
    if max_row(M) > 12:  # wide: restrictions in TMA-CSR when padded, coarse A in SELL-32
        return amgb.FMT_TMACSR if role == "R" and sell_padding(M) > 1.05 and not tcsr_wide(M) else amgb.FMT_SELL
    return amgb.FMT_TMACSR if sell_padding(M) > 1.15 and not tcsr_wide(M) else amgb.FMT_TMA


def max_row(M):
    return int(lens(M).max()) if M.nrows else 0


def tcsr_wide(M):
    # two stages of the largest 256-row tile's entries (12 B) + row pointers
    te = 4
    for r0 in range(0, M.nrows, 256):
        e0, e1 = int(M.ptr[r0]), int(M.ptr[min(r0 + 256, M.nrows)])
        te = max(te, ((e1 - (e0 & ~3)) + 3) & ~3)
    stage = (te * 12 + (256 + 8) * 4 + 15) & ~15
    return 2 * stage + 64 > 227 * 1024


def tcsr_index_cap(M):
    # distinct values a TMA-CSR store can index: its table (8 B per value) shares the
    # 227 KB of shared memory with two stages of 2-byte indices (amgb.cu index_store)
    te = 4
    for r0 in range(0, M.nrows, 256):
        e0, e1 = int(M.ptr[r0]), int(M.ptr[min(r0 + 256, M.nrows)])
        te = max(te, ((e1 - (e0 & ~3)) + 3) & ~3, ((e1 - (e0 & ~15)) + 15) & ~15)
    te = (te + 15) & ~15
    stage = (te * 6 + (256 + 8) * 4 + 15) & ~15
    return min(65536, max(256, (227 * 1024 - 64 - 2 * stage - 256) // 8))


def tma_wide(M):
    # a forced TMA store falls back to SELL-32 when two stages of a 256-row tile
    # do not fit the 227 KB of shared memory (pick_format)
    return 2 * 256 * 12 * max(max_row(M), 1) + 64 > 227 * 1024


def setup_pair(gen, n, kw, fmt, monkeypatch):
    for k in ("AMGB_FORMAT", "AMGB_NO_DICT"):
        monkeypatch.delenv(k, raising=False)
    for k, v in FORMATS[fmt].items():
        monkeypatch.setenv(k, v)
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, **kw)
    ok = {k: w for k, w in kw.items() if k != "reorder"}
    o = oracle.Hierarchy(oracle.Csr(p, c, v), **okw(ok))
    return h, o


@pytest.mark.parametrize("fmt", list(FORMATS))
@pytest.mark.parametrize("gen,n,kw", CASES)
def test_fused_kernels_per_row(gen, n, kw, fmt, monkeypatch):
    h, o = setup_pair(gen, n, kw, fmt, monkeypatch)
    assert h.nlevels == o.nlevels >= 2
    relax = kw.get("relax", "spai0")
    cheb = relax == "chebyshev"
    rng = np.random.default_rng(synth.SEED_VEC)
    for l in range(h.nlevels - 1):
        A, P, R = o.matrix(l, "A"), o.matrix(l, "P"), o.matrix(l, "R")
        info = h.level_info(l)
        # the store is in the format this case is about
        for key, M, role in (("fmt_A", A, "A"), ("fmt_P", P, "P"), ("fmt_R", R, "R")):
            assert info[key] == expected_fmt(fmt, M, role), (l, key, info["formats"])
        if fmt == "tma_explicit":
            assert info["dict_slices_A"] == 0
        n_l, nc = A.nrows, P.ncols
        x = rng.standard_normal(n_l)
        fl = rng.standard_normal(n_l)
        e = rng.standard_normal(nc)
        t = rng.standard_normal(n_l)

        # plain SpMV / residual (amg_level_op)
        for op, M, vin, g in ((amgb.OP_SPMV_A, A, x, None), (amgb.OP_SPMV_P, P, e, None),
                              (amgb.OP_SPMV_R, R, t, None), (amgb.OP_RESIDUAL, A, x, fl)):
            y = host(h.level_op(l, op, x=dev(vin), f=dev(g) if g is not None else None, ny=M.nrows))
            ref = oracle.spmv(M, vin)
            if g is not None:
                ref = g - ref
            check_rows(y, ref, row_bound(M, vin, 0.0 if g is None else g), f"level {l} op {op}")

        # a5 general prolongation x += P e
        xo = dev(x)
        h.level_op_ex(l, amgb.OP_PROL_ADD, in0=dev(e), out0=xo)
        check_rows(host(xo), x + oracle.spmv(P, e), row_bound(P, e, x), f"level {l} prolong add")

        if not cheb:
            m = o.smoother(l)
            mf = m * fl  # one IEEE product, as the kernels form m_j f_j
            # a1: t = f - A (m o f), with m o f formed in the gather, and given
            y = empty(n_l)
            h.level_op_ex(l, amgb.OP_RES0, in0=dev(fl), out0=y)
            ref = fl - oracle.spmv(A, mf)
            check_rows(host(y), ref, row_bound(A, mf, fl), f"level {l} res0")
            y = empty(n_l)
            h.level_op_ex(l, amgb.OP_RES0_MF, in0=dev(fl), in1=dev(mf), out0=y)
            check_rows(host(y), ref, row_bound(A, mf, fl), f"level {l} res0 (mf)")
            # a5 after the zero-start sweep: x = m o f + P e
            y = empty(n_l)
            h.level_op_ex(l, amgb.OP_PROL0, in0=dev(e), in1=dev(fl), out0=y)
            ref = mf + oracle.spmv(P, e)
            check_rows(host(y), ref, row_bound(P, e, mf), f"level {l} prolong0")
            y = empty(n_l)
            h.level_op_ex(l, amgb.OP_PROL0_MF, in0=dev(e), in1=dev(mf), out0=y)
            check_rows(host(y), ref, row_bound(P, e, mf), f"level {l} prolong0 (mf)")
            # a6: one sweep from a non-zero x, fused (f, x')
            y = empty(n_l)
            rho = h.level_op_ex(l, amgb.OP_RELAX_RHO, in0=dev(x), in1=dev(fl), out0=y)
            ref = o.relax(l, fl, x)
            r_ref = fl - oracle.spmv(A, x)
            b = np.abs(m) * row_bound(A, x, fl) + 4 * U * (np.abs(x) + np.abs(m * r_ref))
            yh = host(y)
            check_rows(yh, ref, b, f"level {l} relax+rho")
            assert abs(rho - np.dot(fl, ref)) <= dot_bound(fl, ref, 0.0, b), (l, rho)
            # plain relax (amg_level_op) against the oracle's smoother call, per row
            y2 = host(h.level_op(l, amgb.OP_RELAX, x=dev(x), f=dev(fl), ny=n_l))
            check_rows(y2, ref, b, f"level {l} relax")
            # a2: f_c = R t and the next level's m_c o f_c (bitwise one product)
            if h.level_info(l + 1)["is_coarsest"]:
                continue
            mc = o.smoother(l + 1)
            yc, mfc = empty(nc), empty(nc)
            h.level_op_ex(l, amgb.OP_RESTRICT_MF, in0=dev(t), out0=yc, out1=mfc)
            ych = host(yc)
            check_rows(ych, oracle.spmv(R, t), row_bound(R, t), f"level {l} restrict (+mf)")
            assert np.array_equal(host(mfc), mc * ych), f"level {l} m_c o f_c"
        else:
            # Chebyshev: each of the K steps of one smoother call, per row, from
            # the GPU's own previous step (so each kernel is checked alone)
            K = h.prm.cheb_degree
            rows = np.repeat(np.arange(n_l), lens(A).astype(np.int64))
            d = np.zeros(n_l)
            d[rows[A.col == rows]] = A.val[A.col == rows]
            xg = x.copy()
            pg = np.zeros(n_l)
            alpha_prev = 0.0
            for k in range(K):
                xd, pd = empty(n_l), dev(pg)
                dot = h.level_op_ex(l, amgb.OP_CHEB_STEP, in0=dev(xg), in1=dev(fl), out0=xd, out1=pd, scalar=k)
                x_ref, p_ref, alpha_k = o.cheb_step(l, k, fl, xg, pg, alpha_prev)
                beta_k = alpha_k * o.smoother(l)[2] - 1.0 if k > 0 else 0.0
                r_ref = (fl - oracle.spmv(A, xg)) / np.abs(d)
                b_r = row_bound(A, xg, fl) / np.abs(d) + 2 * U * np.abs(r_ref)
                b_p = abs(alpha_k) * b_r + 3 * U * (np.abs(alpha_k * r_ref) + np.abs(beta_k * pg))
                b_x = b_p + 2 * U * (np.abs(xg) + np.abs(p_ref))
                ph, xh = host(pd), host(xd)
                check_rows(ph, p_ref, b_p, f"level {l} cheb step {k} p")
                check_rows(xh, x_ref, b_x, f"level {l} cheb step {k} x")
                assert abs(dot - np.dot(fl, x_ref)) <= dot_bound(fl, x_ref, 0.0, b_x), (l, k, dot)
                xg, pg, alpha_prev = xh, ph, alpha_k
            # the K steps compose to the oracle's smoother call (norm bar)
            ref = o.relax(l, fl, x)
            y = host(h.level_op(l, amgb.OP_RELAX, x=dev(x), f=dev(fl), ny=n_l))
            assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref), l
            assert np.array_equal(y, xg), "OP_RELAX == K chained CHEB_STEP launches"

    # level 0: the CG direction (a7) and the CG update (a8)
    A = o.matrix(0, "A")
    n0 = A.nrows
    z, pv = rng.standard_normal(n0), rng.standard_normal(n0)
    beta = 0.37
    pn, q = empty(n0), empty(n0)
    sigma = h.level_op_ex(0, amgb.OP_CG_DIR, in0=dev(z), in1=dev(pv), out0=pn, out1=q, scalar=beta)
    p_ref = z + beta * pv
    b_p = 2 * U * (np.abs(z) + np.abs(beta * pv))
    pnh, qh = host(pn), host(q)
    check_rows(pnh, p_ref, b_p, "cg dir p'")
    q_ref = oracle.spmv(A, p_ref)
    b_q = 8 * (lens(A) + 2) * U * absdot(A, np.abs(z) + np.abs(beta * pv))
    check_rows(qh, q_ref, b_q, "cg dir q")
    assert abs(sigma - np.dot(p_ref, q_ref)) <= dot_bound(p_ref, q_ref, b_p, b_q), sigma
    if not cheb:
        m0 = o.smoother(0)
        xv, rv, qv = rng.standard_normal(n0), rng.standard_normal(n0), rng.standard_normal(n0)
        alpha = -0.61
        xd, rd, mfd = dev(xv), dev(rv), empty(n0)
        res = h.level_op_ex(0, amgb.OP_CG_UPDATE, in0=dev(pv), in1=dev(qv), out0=xd, out1=rd, out2=mfd,
                            scalar=alpha)
        xh, rh = host(xd), host(rd)
        check_rows(xh, xv + alpha * pv, 2 * U * (np.abs(xv) + np.abs(alpha * pv)), "cg update x")
        r_ref = rv - alpha * qv
        b_r = 2 * U * (np.abs(rv) + np.abs(alpha * qv))
        check_rows(rh, r_ref, b_r, "cg update r")
        assert np.array_equal(host(mfd), m0 * rh), "cg update m o r"
        rr = np.dot(r_ref, r_ref)
        assert abs(res * res - rr) <= dot_bound(r_ref, r_ref, b_r, b_r) + 4 * U * rr, (res, rr)


@pytest.mark.parametrize("fmt", ["auto", "sell", "tma_explicit", "tmacsr"])
def test_vcycle_and_solve_per_format(fmt, monkeypatch):
    """The whole V-cycle (1e-12) and a converged CG solve (iterations +-1, x within
    1e-8 at equal count) in each format at >= 65,536 rows."""
    h, o = setup_pair("poisson", 41, {}, fmt, monkeypatch)
    p, c, v, f = synth.problem("poisson", 41)
    r = synth.random_vector(len(f))
    z = host(h.precond(dev(r)))
    ref = o.precond(r)
    assert np.linalg.norm(z - ref) <= 1e-12 * np.linalg.norm(ref)
    x, iters, rel, st = h.solve(dev(f), tol=1e-8, maxiter=100)
    oc = oracle.cg(oracle.Csr(p, c, v), f, tol=1e-8, maxiter=100, hier=o)
    assert st == amgb.OK and abs(iters - oc["iters"]) <= 1
    if iters != oc["iters"]:
        x, iters, rel, st = h.solve(dev(f), tol=0.0, maxiter=oc["iters"])
    assert np.linalg.norm(host(x) - oc["x"]) <= 1e-8 * np.linalg.norm(oc["x"])


@pytest.mark.parametrize("tmacsr", [None, "4"])
def test_level1_in_sell_and_tma_under_auto(tmacsr, monkeypatch):
    """88^3 (681,472 rows): level 1 has >= 65,536 rows, so under the default policy
    A0 runs sell_tma, P0 / R0 csr_tma and A1 sell_rows with 2-byte value indices,
    as at 256^3 (AMGB_TMACSR=4: A1 in csr_tma with 2-byte indices and the table in
    shared memory, when its distinct values fit); every op of levels 0-1 per row
    against the oracle."""
    for k in ("AMGB_FORMAT", "AMGB_NO_DICT", "AMGB_TMACSR"):
        monkeypatch.delenv(k, raising=False)
    if tmacsr:
        monkeypatch.setenv("AMGB_TMACSR", tmacsr)
    p, c, v, f = synth.problem("poisson", 88)
    h = amgb.setup(p, c, v)
    o = oracle.Hierarchy(oracle.Csr(p, c, v))
    i1 = h.level_info(1)
    assert i1["rows"] >= 65536
    assert h.level_info(0)["fmt_A"] == amgb.FMT_TMA and h.level_info(0)["fmt_P"] == amgb.FMT_TMACSR
    assert h.level_info(0)["fmt_R"] == amgb.FMT_TMACSR
    A1 = o.matrix(1, "A")
    assert 256 < len(np.unique(A1.val)) <= tcsr_index_cap(A1) and sell_padding(A1) > 1.05
    assert i1["fmt_A"] == (amgb.FMT_TMACSR if tmacsr else amgb.FMT_SELL) and i1["vidx_A"] == 2
    rng = np.random.default_rng(7)
    for l in (0, 1):
        A, P, R = o.matrix(l, "A"), o.matrix(l, "P"), o.matrix(l, "R")
        m = o.smoother(l)
        fl = rng.standard_normal(A.nrows)
        x = rng.standard_normal(A.nrows)
        e = rng.standard_normal(P.ncols)
        t = rng.standard_normal(A.nrows)
        mf = m * fl
        y = empty(A.nrows)
        h.level_op_ex(l, amgb.OP_RES0_MF, in0=dev(fl), in1=dev(mf), out0=y)
        check_rows(host(y), fl - oracle.spmv(A, mf), row_bound(A, mf, fl), f"l{l} res0")
        y = empty(A.nrows)
        h.level_op_ex(l, amgb.OP_PROL0_MF, in0=dev(e), in1=dev(mf), out0=y)
        check_rows(host(y), mf + oracle.spmv(P, e), row_bound(P, e, mf), f"l{l} prolong0")
        y = empty(A.nrows)
        rho = h.level_op_ex(l, amgb.OP_RELAX_RHO, in0=dev(x), in1=dev(fl), out0=y)
        ref = o.relax(l, fl, x)
        b = np.abs(m) * row_bound(A, x, fl) + 4 * U * (np.abs(x) + np.abs(m * (fl - oracle.spmv(A, x))))
        check_rows(host(y), ref, b, f"l{l} relax")
        assert abs(rho - np.dot(fl, ref)) <= dot_bound(fl, ref, 0.0, b)
        yc, mfc = empty(P.ncols), empty(P.ncols)
        h.level_op_ex(l, amgb.OP_RESTRICT_MF, in0=dev(t), out0=yc, out1=mfc)
        ych = host(yc)
        check_rows(ych, oracle.spmv(R, t), row_bound(R, t), f"l{l} restrict")
        assert np.array_equal(host(mfc), o.smoother(l + 1) * ych)


@pytest.mark.parametrize("k", [4, 8])
@pytest.mark.parametrize("gen,n,kw", [("poisson", 41, {}), ("varcoef", 41, {"relax": "chebyshev"})])
def test_batched_columns_match_oracle(gen, n, kw, k, monkeypatch):
    """amg_solve_batched on the TMA / SELL store (>= 65,536 rows) against the
    oracle, column by column: iterations +-1, x within 1e-8 at equal count."""
    for key in ("AMGB_FORMAT", "AMGB_NO_DICT"):
        monkeypatch.delenv(key, raising=False)
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, **kw)
    assert h.level_info(0)["fmt_A"] == amgb.FMT_TMA
    A = oracle.Csr(p, c, v)
    hier = oracle.Hierarchy(A, **okw(kw))
    rng = np.random.default_rng(100 + k)
    F = np.stack([f] + [rng.standard_normal(len(f)) for _ in range(k - 1)])
    X, iters, rels, st = h.solve_batched(dev(F), tol=1e-8, maxiter=200)
    Xh = host(X)
    assert st == amgb.OK
    for j in range(k):
        oc = oracle.cg(A, F[j], tol=1e-8, maxiter=200, hier=hier)
        assert abs(int(iters[j]) - oc["iters"]) <= 1, (j, iters[j], oc["iters"])
        if iters[j] != oc["iters"]:  # compare at equal iteration count (§8c)
            oc = oracle.cg(A, F[j], tol=0.0, maxiter=int(iters[j]), hier=hier)
        assert np.linalg.norm(Xh[j] - oc["x"]) <= 1e-8 * np.linalg.norm(oc["x"]), j


@pytest.mark.parametrize("gen,n,kw", [("poisson", 48, {}), ("convdiff", 48, {"relax": "damped_jacobi",
                                                                             "solver": "bicgstab"}),
                                      ("poisson", 41, {"AMGB_FORMAT": "sell"})])
def test_value_indexed_store_is_bitwise_the_plain_store(gen, n, kw, monkeypatch):
    """Value-indexed storage (the default: a table of the distinct values + 1- or
    2-byte indices, amgb.cu value_index) is lossless: every level op, the V-cycle
    and the whole solve are bitwise those of the fp64-array store (AMGB_VIDX=0)."""
    for k in ("AMGB_FORMAT", "AMGB_NO_DICT", "AMGB_VIDX"):
        monkeypatch.delenv(k, raising=False)
    kw = dict(kw)
    if "AMGB_FORMAT" in kw:
        monkeypatch.setenv("AMGB_FORMAT", kw.pop("AMGB_FORMAT"))
    p, c, v, f = synth.problem(gen, n)
    hv = amgb.setup(p, c, v, **kw)  # the default
    monkeypatch.setenv("AMGB_VIDX", "0")
    hp = amgb.setup(p, c, v, **kw)
    i0 = hv.level_info(0)
    assert i0["vidx_A"] == 1 and hp.level_info(0)["vidx_A"] == 0  # constant coefficients: <= 256 values
    assert i0["dev_bytes"] < hp.level_info(0)["dev_bytes"]
    rng = np.random.default_rng(5)
    for l in range(hv.nlevels - 1):
        inf = hv.level_info(l)
        x = dev(rng.standard_normal(inf["rows"]))
        e = dev(rng.standard_normal(inf["cols_P"]))
        for op, vin, ny in ((amgb.OP_SPMV_A, x, inf["rows"]), (amgb.OP_SPMV_P, e, inf["rows"]),
                            (amgb.OP_SPMV_R, x, inf["cols_P"])):
            assert np.array_equal(host(hv.level_op(l, op, x=vin, ny=ny)), host(hp.level_op(l, op, x=vin, ny=ny)))
    r = dev(synth.random_vector(len(f)))
    assert np.array_equal(host(hv.precond(r)), host(hp.precond(r)))
    xv, itv, relv, stv = hv.solve(dev(f), tol=1e-8, maxiter=200)
    xp, itp, relp, stp = hp.solve(dev(f), tol=1e-8, maxiter=200)
    assert stv == stp == amgb.OK and itv == itp and relv == relp
    assert np.array_equal(host(xv), host(xp))
