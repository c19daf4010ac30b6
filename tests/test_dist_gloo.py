"""World-size-2 CPU tests (gloo) of the N>1 host logic: unique-id broadcast, per-rank plans
from the library's planner agreeing across ranks, and the straddler exchange protocol
(row per rank, summed in rank order) reproducing the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        globals()[fn_name](rank, world)
        q.put((rank, "ok"))
    except BaseException as e:  # noqa
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
    for r in range(world):
        assert res[r] == "ok", res[r]


# ------------------------------------------------------------------ rank bodies
def body_host_allgather(rank, world):
    """The bootstrap callback lamb_create_with_allgather calls (IPC handles, table hash):
    rank j's bytes land at offset j * nbytes on every rank; a size mismatch reports failure."""
    import ctypes
    from paper_2402_15627_b200 import lamb
    fn = lamb._pg_allgather(dist.group.WORLD)
    nb = 192   # three cudaIpcMemHandle_t
    send = (ctypes.c_uint8 * nb)(*[(rank * 31 + i) % 256 for i in range(nb)])
    recv = (ctypes.c_uint8 * (nb * world))()
    cfn = ctypes.cast(fn, ctypes.c_void_p)
    call = lamb._ALLGATHER_FN(cfn.value)
    assert call(ctypes.addressof(send), ctypes.addressof(recv), nb, None) == 0
    got = bytes(recv)
    for j in range(world):
        assert got[j * nb:(j + 1) * nb] == bytes((j * 31 + i) % 256 for i in range(nb))
    # ranks passing different sizes: every rank must see the failure, none may hang
    nb2 = 8 + rank
    send2 = (ctypes.c_uint8 * nb2)()
    recv2 = (ctypes.c_uint8 * (nb2 * world))()
    lamb._ag_errors.clear()
    assert call(ctypes.addressof(send2), ctypes.addressof(recv2), nb2, None) == 1
    assert lamb._ag_errors and "bootstrap bytes" in lamb._ag_errors[-1]   # reported, not swallowed


def body_unique_id(rank, world):
    from paper_2402_15627_b200 import lamb
    uid = lamb.broadcast_unique_id(dist.group.WORLD, rank, 0)
    assert len(uid) == 128
    out = [None] * world
    dist.all_gather_object(out, uid)
    assert all(u == out[0] for u in out) and any(out[0])


def body_plans_agree(rank, world):
    from paper_2402_15627_b200 import lamb
    for name in ("toy", "gpt1.3b", "530b_stress"):
        wl = W.get(name)
        numels = [t.numel for t in wl.tensors]
        pv = lamb.host_plan(numels, world, rank, wl.cap)
        mine = (pv.tensor_off.tolist(), pv.buckets.tolist(), pv.straddlers.tolist(), pv.segments.tolist())
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        assert all(a[0] == allp[0][0] and a[1] == allp[0][1] and a[2] == allp[0][2] for a in allp)
        cover = {}
        for r, a in enumerate(allp):
            for (i, soff, toff, ln) in a[3]:
                cover.setdefault(i, []).append((toff, ln))
        for i, n in enumerate(numels):
            parts = sorted(cover[i])
            assert parts[0][0] == 0 and sum(ln for _, ln in parts) == n
            assert all(parts[k][0] + parts[k][1] == parts[k + 1][0] for k in range(len(parts) - 1))
        strad = [i for i, p in cover.items() if len(p) > 1]
        assert sorted(strad) == allp[0][2]


def body_straddler_exchange(rank, world):
    """Each rank updates only its segments; straddler partials travel as one row per rank
    (slot = index in the global straddler list), summed in rank order 0..D-1."""
    import torch
    from paper_2402_15627_b200 import lamb
    rng = np.random.default_rng(4)
    tensors = W.random_table(rng, 25, max_numel=900, p_big=0.2, big=5000)
    wl = W.Workload("x", 60, tensors, W.default_groups(lr=2.0 ** -7))
    numels = [t.numel for t in tensors]
    pv = lamb.host_plan(numels, world, rank, 4096)
    assert len(pv.straddlers) > 0
    slot = {int(t): k for k, t in enumerate(pv.straddlers)}
    ref = oracle.OracleRun(wl, world_size=world, mode=oracle.PER_RANK)
    mine = {}
    row = np.zeros((len(pv.straddlers), 2))
    local = {}
    for (i, soff, toff, ln) in pv.segments.tolist():
        g = ref.grads(i, 1)[toff:toff + ln]
        w = ref.w[i][toff:toff + ln].copy()
        m = np.zeros(ln); v = np.zeros(ln)
        u = oracle.moments_and_update(w, m, v, g, wl.groups[tensors[i].group], 1)
        mine[i] = (toff, w, u)
        w2, u2 = oracle.sumsq(w), oracle.sumsq(u)
        if i in slot:
            row[slot[i]] = (w2, u2)
        else:
            local[i] = (w2, u2)
    rows = [torch.zeros_like(torch.from_numpy(row)) for _ in range(world)]
    dist.all_gather(rows, torch.from_numpy(row))
    ref.step(1)
    for i, (toff, w, u) in mine.items():
        if i in slot:
            w2 = sum(float(rows[j][slot[i], 0]) for j in range(world))
            u2 = sum(float(rows[j][slot[i], 1]) for j in range(world))
        else:
            w2, u2 = local[i]
        grp = wl.groups[tensors[i].group]
        r = oracle.trust_ratio(np.sqrt(w2), np.sqrt(u2), grp.adapt)
        assert r == pytest.approx(ref.stats[i][2], rel=1e-13)
        oracle.apply(w, u, oracle.f32(grp.lr), r)
        assert np.allclose(w, ref.w[i][toff:toff + len(w)], rtol=1e-13, atol=1e-17)


def test_unique_id_broadcast_gloo():
    _run("body_unique_id")


def test_plans_agree_across_ranks_gloo():
    _run("body_plans_agree")


def test_straddler_exchange_protocol_gloo():
    _run("body_straddler_exchange")


def test_host_allgather_bootstrap():
    _run("body_host_allgather")
