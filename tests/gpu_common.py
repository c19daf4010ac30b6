"""Helpers for the GPU parity tests: run the CUDA path through the C-ABI and compare with
the oracle per tensor.  Tolerances are DESIGN.md §3 "Comparison rule" (north_star: 1e-5
relative / 1e-6 absolute after 1 step, 1e-4 after 10 steps), plus the per-step update check
(DESIGN.md §3 "Update check"): the state tolerance's 1e-6 absolute floor is ~1-7 % of one
LAMB step, so on its own it cannot see a pass B that applies a slightly wrong u."""
from __future__ import annotations

import numpy as np

import oracle
import workloads as W


def spec_of(wl):
    return [(t.init, t.gexp) for t in wl.tensors]


def run_gpu(wl, D=1, rank=0, steps=1, mode=oracle.PER_RANK, device=0, cap=None, groups=None,
            comm_mode=1, unique_id=None, timing=False, snapshot=True):
    from paper_2402_15627_b200 import lamb
    groups = groups if groups is not None else wl.groups
    L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], groups, world_size=D, rank=rank,
                  device=device, comm_mode=comm_mode, bucket_cap=cap if cap is not None else wl.cap,
                  unique_id=unique_id, timing=timing)
    spec = spec_of(wl)
    L.synth_init(spec, wl.seed)
    rterm = oracle.rank_term(mode, rank)
    for t in range(1, steps + 1):
        L.synth_grads(spec, wl.seed, rterm, t)
        if t == steps and snapshot:
            L.w_prev = snapshot_w(L)       # for the per-step update check in compare_state
        L.step(t)
    return L


def snapshot_w(L, ids=None):
    """This rank's fp32 master pieces {tensor: [(tensor_off, values)]} as they are now (host
    copies).  Taken right before a step, it lets compare_state check that step's update."""
    lm = lamb_mod()
    if ids is None:
        return shard_to_tensors(L, L.get_state(lm.LAMB_BUF_W))
    ids = set(ids)
    buf = L.state_buffer(lm.LAMB_BUF_W)
    out = {}
    for (i, soff, toff, ln) in L.plan.segments.tolist():
        if i in ids:
            out.setdefault(i, []).append((toff, buf[soff:soff + ln].cpu().numpy()))
    return out


def update_excess(gw, gw_prev, ow, ow_prev, dmax, rtol=1e-5):
    """Per-step update check: dw_gpu = w_new - w_prev of the fp32 master (exact
    in double) against the oracle's dw = -lr ratio u of the same step.  Allowed per element:
    1 ulp of the fp32 w (pass B rounds w - s u once: <= 0.5 ulp, and the binade may change),
    rtol |dw_orc| (u and the ratio carry ~1e-7 relative error) and 1e-6 of the tensor's largest
    |dw_orc| (u near zero by cancellation).  A pass B that drops the decay term from u or scales
    the update by 1.005 exceeds it by > 3x at lr 2^-10 and > 20x at lr 2^-7 (CPU emulation of
    the kernel arithmetic; GPU mutants recorded in DESIGN.md §3).  Returns max(|err| / allowed)."""
    worst = 0.0
    for lo in range(0, len(gw), 1 << 24):          # bounded host memory on 2^31-element tensors
        hi = lo + (1 << 24)
        g1 = np.asarray(gw[lo:hi], np.float32)
        g0 = np.asarray(gw_prev[lo:hi], np.float32)
        dg = g1.astype(np.float64) - g0.astype(np.float64)
        do = np.asarray(ow[lo:hi], np.float64) - np.asarray(ow_prev[lo:hi], np.float64)
        ulp = np.spacing(np.maximum(np.abs(g1), np.abs(g0))).astype(np.float64)
        allowed = ulp + rtol * np.abs(do) + 1e-6 * dmax
        worst = max(worst, float(np.max(np.abs(dg - do) / allowed)))
    return worst


def shard_to_tensors(L, arr, ids=None):
    """Per-tensor pieces (tensor_off -> values) of this rank's shard array."""
    out = {}
    for (i, soff, toff, ln) in L.plan.segments.tolist():
        if ids is not None and i not in ids:
            continue
        out.setdefault(i, []).append((toff, arr[soff:soff + ln]))
    return out


def tol(steps):
    return 1e-5 if steps <= 1 else 1e-4


def compare_state(L, orc: oracle.OracleRun, steps: int, ids=None, check_params=True, w_prev=None):
    """Compare this rank's pieces of w, m, v (and params/ratios) with the oracle; with the GPU's
    master before the last step (`w_prev`, default L.w_prev from run_gpu / snapshot_w) also
    that step's update dw per element (update_excess)."""
    rtol = tol(steps)
    if w_prev is None:
        w_prev = getattr(L, "w_prev", None)
    upd_worst = 0.0
    lm = lamb_mod()
    if ids is None:
        ids = set(orc.ids)
        w, m, v = (L.get_state(k) for k in (lm.LAMB_BUF_W, lm.LAMB_BUF_M, lm.LAMB_BUF_V))
        pw, pm, pv = shard_to_tensors(L, w, ids), shard_to_tensors(L, m, ids), shard_to_tensors(L, v, ids)
    else:   # large configs: fetch only the checked segments from the device
        ids = set(ids)
        pw, pm, pv = {}, {}, {}
        bufs = [L.state_buffer(k) for k in (lm.LAMB_BUF_W, lm.LAMB_BUF_M, lm.LAMB_BUF_V)]
        for (i, soff, toff, ln) in L.plan.segments.tolist():
            if i in ids:
                for d, buf in zip((pw, pm, pv), bufs):
                    d.setdefault(i, []).append((toff, buf[soff:soff + ln].cpu().numpy()))
    w2, u2, ratio = L.tensor_stats()
    params = L.param_buffer().view(__import__("torch").int16).cpu().numpy().view(np.uint16) if check_params else None
    worst = 0.0
    for i in ids:
        if i not in pw:
            continue
        for (toff, gw), (_, gm), (_, gv) in zip(pw[i], pm[i], pv[i]):
            n = len(gw)
            ow, om, ov = orc.w[i][toff:toff + n], orc.m[i][toff:toff + n], orc.v[i][toff:toff + n]
            ew = np.abs(gw - ow) - (1e-6 + rtol * np.abs(ow))
            em = np.abs(gm - om) - (1e-6 * np.max(np.abs(orc.m[i])) + rtol * np.abs(om))
            ev = np.abs(gv - ov) - (1e-6 * np.max(np.abs(orc.v[i])) + rtol * np.abs(ov))
            for name, e in (("w", ew), ("m", em), ("v", ev)):
                if np.any(e > 0):
                    k = int(np.argmax(e))
                    raise AssertionError(f"tensor {i} {name}[{toff + k}] out of tolerance: "
                                         f"gpu={[gw, gm, gv][['w','m','v'].index(name)][k]!r} "
                                         f"orc={[ow, om, ov][['w','m','v'].index(name)][k]!r}")
            # reported: relative error where it means something (|w| >= 1e-3; smaller |w| are
            # governed by the 1e-6 absolute term) — the pass/fail test is the tolerance above
            big = np.abs(ow) >= 1e-3
            if np.any(big):
                worst = max(worst, float(np.max(np.abs(gw[big] - ow[big]) / np.abs(ow[big]))))
            if w_prev is not None and i in orc.w_prev:
                prev = dict((o, a) for o, a in w_prev.get(i, []))
                assert toff in prev, f"tensor {i}: no pre-step snapshot of the piece at {toff}"
                dmax = float(np.max(np.abs(orc.w[i] - orc.w_prev[i])))
                x = update_excess(gw, prev[toff], ow, orc.w_prev[i][toff:toff + n], dmax)
                if x > 1.0:
                    raise AssertionError(f"tensor {i}: per-step update dw out of tolerance "
                                         f"(max |err|/allowed = {x:.3g})")
                upd_worst = max(upd_worst, x)
            if check_params:
                off = int(L.plan.tensor_off[i]) + toff
                assert np.array_equal(params[off:off + n], oracle.bf16_rne_bits(gw.astype(np.float64))), \
                    f"tensor {i}: params != bf16_rne(w_gpu)"   # H11
        if not np.isnan(ratio[i]):
            wn, un, r = orc.stats[i]
            assert abs(ratio[i] - r) <= rtol * abs(r) + 1e-7, (i, ratio[i], r)
            assert abs(np.sqrt(w2[i]) - wn) <= 1e-6 * max(wn, 1e-30) + 1e-12, (i, np.sqrt(w2[i]), wn)
    L.update_worst = upd_worst      # reported by tests (max |err|/allowed of the update check)
    return worst


def lamb_mod():
    from paper_2402_15627_b200 import lamb
    return lamb
