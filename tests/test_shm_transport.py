"""The host shared-memory TEST transport of the multi-process path (CPU, no
GPU): 3 processes run amg_shm_selftest -- three personalised all-to-all rounds
(empty, small and 1 MB segments) through POSIX shared memory, every segment
checked by its receiver -- and a missing peer turns into an error after the
timeout instead of a hang (AMGB_NCCL_TIMEOUT_S)."""
import multiprocessing as mp
import os
import secrets

import pytest


def _worker(tag, rank, nranks, q):
    os.environ["AMGB_NCCL_TIMEOUT_S"] = "20"
    import paper_1811_05704_b200 as amgb
    try:
        amgb.shm_selftest(tag, rank, nranks)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, str(e)))


def _run(nranks, launched):
    tag = secrets.token_bytes(128)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(tag, r, nranks, q)) for r in range(launched)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


def test_shm_alltoallv_three_ranks():
    out = _run(3, 3)
    assert out == {0: "ok", 1: "ok", 2: "ok"}, out


def test_shm_missing_peer_times_out(monkeypatch):
    monkeypatch.setenv("AMGB_NCCL_TIMEOUT_S", "2")
    import paper_1811_05704_b200 as amgb
    with pytest.raises(amgb.AmgError) as ei:
        amgb.shm_selftest(secrets.token_bytes(128), 0, 2)  # rank 1 never comes
    assert ei.value.code == amgb.E_NCCL and "timeout" in str(ei.value)
