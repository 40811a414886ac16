"""Multi-GPU host logic (row partition, ghost renumbering, halo plans) through
the C ABI on CPU: host-only handles (device = -1), "virtual ranks" in one
process and a world_size-2 gloo run with one rank per process.  A distributed
mat-vec emulated from the exported local matrices and plans must equal the
global one bit for bit (row sums keep the global column order)."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1811_05704_b200 as amgb
import synth


def csr(ptr, col, val, ncols):
    return sp.csr_matrix((val, col, ptr), shape=(len(ptr) - 1, ncols))


def global_levels(h):
    """Global A, P, R per level from the host export of a host-only handle."""
    out = []
    for l in range(h.nlevels):
        e = h.export_level(l)
        inf = h.level_info(l)
        n = inf["rows"]
        lv = {"A": csr(*e["A"], n)}
        if not inf["is_coarsest"]:
            lv["P"] = csr(*e["P"], inf["cols_P"])
            lv["R"] = csr(*e["R"], n)
        out.append(lv)
    return out


def to_global_cols(col, row0, nloc, ghost_global, replicated=False):
    col = np.asarray(col, np.int64)
    if replicated:
        return col
    return np.where(col < nloc, col + row0, ghost_global[np.maximum(col - nloc, 0)])


CASES = [("poisson", 20, 2), ("poisson", 20, 3), ("poisson_perm", 14, 4), ("convdiff", 16, 3),
         ("varcoef", 16, 2)]


@pytest.mark.parametrize("gen,n,nranks", CASES)
def test_partition_reconstructs_global(gen, n, nranks):
    p, c, v, f = synth.problem(gen, n)
    kw = {"relax": "chebyshev"} if gen == "varcoef" else {}
    h = amgb.setup_dist(p, c, v, nranks=nranks, rank=-1, gather_below=300, device=-1,
                        coarse_enough=40, **kw)
    g = global_levels(h)
    di = h.dist_info()
    lg = di["first_replicated"]
    assert 1 <= lg <= h.nlevels - 1
    assert di["row_starts"][0] == 0 and di["row_starts"][-1] == len(f)
    exports = {(r, l): h.dist_export(r, l) for r in range(nranks) for l in range(h.nlevels)}
    for l in range(h.nlevels):
        owned = np.zeros(g[l]["A"].shape[0], int)
        for r in range(nranks):
            e = exports[(r, l)]
            inf = e["info"]
            if l >= lg:
                assert inf["replicated"] == 1 and inf["ghosts"] == 0
                assert (csr(*e["A"], g[l]["A"].shape[1]) != g[l]["A"]).nnz == 0
                continue
            row0, row1 = inf["row0"], inf["row1"]
            owned[row0:row1] += 1
            nloc = row1 - row0
            gg = e["ghost_global"]
            assert np.all(np.diff(gg) > 0) and not np.any((gg >= row0) & (gg < row1))
            # A rows: same values in the same (global) order
            Ag = g[l]["A"]
            ptr, col, val = e["A"]
            assert np.array_equal(ptr, Ag.indptr[row0:row1 + 1] - Ag.indptr[row0])
            seg = slice(Ag.indptr[row0], Ag.indptr[row1])
            assert np.array_equal(to_global_cols(col, row0, nloc, gg), Ag.indices[seg])
            assert np.array_equal(val, Ag.data[seg])
            if "P" in e:
                Pg, Rg = g[l]["P"], g[l]["R"]
                crow0, crow1 = inf["crow0"], inf["crow1"]
                # P columns: numbering of level l+1 (global when it is replicated)
                ptr, col, val = e["P"]
                nxt = exports[(r, l + 1)]
                rep = bool(nxt["info"]["replicated"])
                cg = to_global_cols(col, nxt["info"]["row0"], nxt["info"]["row1"] - nxt["info"]["row0"],
                                    nxt["ghost_global"], replicated=rep)
                seg = slice(Pg.indptr[row0], Pg.indptr[row1])
                assert np.array_equal(cg, Pg.indices[seg]) and np.array_equal(val, Pg.data[seg])
                ptr, col, val = e["R"]
                seg = slice(Rg.indptr[crow0], Rg.indptr[crow1])
                assert np.array_equal(to_global_cols(col, row0, nloc, gg), Rg.indices[seg])
                assert np.array_equal(val, Rg.data[seg])
            # halo plan: what r receives from q is exactly what q sends to r
            for k, q in enumerate(e["recv_peer"]):
                eq = exports[(int(q), l)]
                j = list(eq["send_peer"]).index(r)
                sidx = eq["send_idx"][eq["send_off"][j]:eq["send_off"][j] + eq["send_cnt"][j]]
                ro, rc = e["recv_off"][k], e["recv_cnt"][k]
                assert rc == eq["send_cnt"][j]
                assert np.array_equal(gg[ro:ro + rc], sidx + eq["info"]["row0"])
        if l < lg:
            assert np.all(owned == 1)  # the row ranges tile the level


def _emulate_exchange(exports, l, vec_global, r):
    """Local vector with ghosts of rank r, built only through the halo plans."""
    e = exports[(r, l)]
    inf = e["info"]
    nloc = inf["row1"] - inf["row0"]
    ext = np.zeros(nloc + inf["ghosts"])
    ext[:nloc] = vec_global[inf["row0"]:inf["row1"]]
    for k, q in enumerate(e["recv_peer"]):
        eq = exports[(int(q), l)]
        j = list(eq["send_peer"]).index(r)
        src = eq["send_idx"][eq["send_off"][j]:eq["send_off"][j] + eq["send_cnt"][j]]
        qv = vec_global[eq["info"]["row0"]:eq["info"]["row1"]]
        ext[nloc + e["recv_off"][k]: nloc + e["recv_off"][k] + e["recv_cnt"][k]] = qv[src]
    return ext


@pytest.mark.parametrize("gen,n,nranks", CASES[:3])
def test_emulated_distributed_matvecs(gen, n, nranks):
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup_dist(p, c, v, nranks=nranks, rank=-1, gather_below=300, device=-1,
                        coarse_enough=40)
    g = global_levels(h)
    lg = h.dist_info()["first_replicated"]
    exports = {(r, l): h.dist_export(r, l) for r in range(nranks) for l in range(h.nlevels)}
    rng = np.random.default_rng(3)
    for l in range(lg):
        x = rng.standard_normal(g[l]["A"].shape[0])
        xc = rng.standard_normal(g[l]["P"].shape[1])
        yA, yR, yP = g[l]["A"] @ x, g[l]["R"] @ x, g[l]["P"] @ xc
        nxt_rep = l + 1 >= lg
        for r in range(nranks):
            e = exports[(r, l)]
            inf = e["info"]
            nloc = inf["row1"] - inf["row0"]
            ext = _emulate_exchange(exports, l, x, r)
            Al = csr(*e["A"], len(ext))
            assert np.array_equal(Al @ ext, yA[inf["row0"]:inf["row1"]])  # bitwise
            Rl = csr(*e["R"], len(ext))
            assert np.array_equal(Rl @ ext, yR[inf["crow0"]:inf["crow1"]])
            xc_ext = xc if nxt_rep else _emulate_exchange(exports, l + 1, xc, r)
            Pl = csr(*e["P"], len(xc_ext))
            assert np.array_equal(Pl @ xc_ext, yP[inf["row0"]:inf["row1"]])


def test_single_rank_and_errors():
    p, c, v, f = synth.poisson3d(12)
    h = amgb.setup_dist(p, c, v, nranks=1, rank=0, device=-1, coarse_enough=50)
    di = h.dist_info()
    assert di["nranks"] == 1 and list(di["row_starts"]) == [0, len(f)]
    with pytest.raises(amgb.AmgError):  # single-level hierarchy cannot be distributed
        amgb.setup_dist(p, c, v, nranks=2, rank=-1, device=-1)
    with pytest.raises(amgb.AmgError):
        amgb.setup_dist(p, c, v, nranks=2, rank=5, device=-1, coarse_enough=50)


# ---------------------------------------------------------------- gloo, 2 ranks

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, c, v, f = synth.problem("poisson", 18)
        h = amgb.setup_dist(p, c, v, nranks=world, rank=rank, gather_below=200, device=-1,
                            coarse_enough=40)
        g = global_levels(h)
        lg = h.dist_info()["first_replicated"]
        ok = True
        for l in range(lg):
            e = h.dist_export(rank, l)
            inf = e["info"]
            nloc = inf["row1"] - inf["row0"]
            x = np.random.default_rng(l).standard_normal(g[l]["A"].shape[0])
            xl = x[inf["row0"]:inf["row1"]]
            ext = np.zeros(nloc + inf["ghosts"])
            ext[:nloc] = xl
            # the halo exchange over gloo, following the plan only
            reqs = []
            for j, peer in enumerate(e["send_peer"]):
                buf = torch.from_numpy(xl[e["send_idx"][e["send_off"][j]:e["send_off"][j] + e["send_cnt"][j]]])
                reqs.append(dist.isend(buf.contiguous(), int(peer)))
            for k, peer in enumerate(e["recv_peer"]):
                buf = torch.zeros(int(e["recv_cnt"][k]), dtype=torch.float64)
                dist.recv(buf, int(peer))
                ext[nloc + e["recv_off"][k]: nloc + e["recv_off"][k] + e["recv_cnt"][k]] = buf.numpy()
            for rq in reqs:
                rq.wait()
            y = csr(*e["A"], len(ext)) @ ext
            ok &= bool(np.array_equal(y, (g[l]["A"] @ x)[inf["row0"]:inf["row1"]]))
            yr = csr(*e["R"], len(ext)) @ ext
            ok &= bool(np.array_equal(yr, (g[l]["R"] @ x)[inf["crow0"]:inf["crow1"]]))
        # dot products: local partial sums, all-reduced
        x = np.random.default_rng(9).standard_normal(len(f))
        st = h.dist_info()["row_starts"]
        part = torch.tensor([float(x[st[rank]:st[rank + 1]] @ x[st[rank]:st[rank + 1]])], dtype=torch.float64)
        dist.all_reduce(part)
        ok &= bool(abs(part.item() - x @ x) <= 1e-12 * (x @ x))
        q.put((rank, ok))
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: True, 1: True}, res
