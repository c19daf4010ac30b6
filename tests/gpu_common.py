"""Helpers for the GPU parity tests: run the CUDA path through the C-ABI and compare with
the oracle per tensor.  Tolerances are DESIGN.md §3 "Comparison rule" (north_star: 1e-5
relative / 1e-6 absolute after 1 step, 1e-4 after 10 steps)."""
from __future__ import annotations

import numpy as np

import oracle
import workloads as W


def spec_of(wl):
    return [(t.init, t.gexp) for t in wl.tensors]


def run_gpu(wl, D=1, rank=0, steps=1, mode=oracle.PER_RANK, device=0, cap=None, groups=None,
            comm_mode=1, unique_id=None, timing=False):
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
        L.step(t)
    return L


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


def compare_state(L, orc: oracle.OracleRun, steps: int, ids=None, check_params=True):
    """Compare this rank's pieces of w, m, v (and params/ratios) with the oracle."""
    rtol = tol(steps)
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
            if check_params:
                off = int(L.plan.tensor_off[i]) + toff
                assert np.array_equal(params[off:off + n], oracle.bf16_rne_bits(gw.astype(np.float64))), \
                    f"tensor {i}: params != bf16_rne(w_gpu)"   # H11
        if not np.isnan(ratio[i]):
            wn, un, r = orc.stats[i]
            assert abs(ratio[i] - r) <= rtol * abs(r) + 1e-7, (i, ratio[i], r)
            assert abs(np.sqrt(w2[i]) - wn) <= 1e-6 * max(wn, 1e-30) + 1e-12, (i, np.sqrt(w2[i]), wn)
    return worst


def lamb_mod():
    from paper_2402_15627_b200 import lamb
    return lamb
