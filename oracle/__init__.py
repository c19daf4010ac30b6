"""CPU oracle for the MegaScale LAMB step.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this package.  The product path (paper_2402_15627_b200/) never imports it and
shares no code with it.  The arithmetic lives in lamb_oracle.c (plain C, double); the
planner in plan.py (plain Python).  See lamb_oracle.c's header for the passages followed
and DESIGN.md §3 for the readings and pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Iterable, List, Optional, Sequence

import numpy as np

from . import plan as plan_mod  # noqa: F401  (re-export)
from .plan import OraclePlan, plan

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lamb_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

REPLICATED, PER_RANK = 0, 1


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -fopenmp, no -ffast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        D, I64, I32, U32, U64 = ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
        P = ctypes.c_void_p
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_gen_word.argtypes = [U64, U32, U32, U32, U32, I64]
        L.orc_gen_word.restype = U32
        L.orc_gen_weights.argtypes = [U64, U32, I32, I64, P]
        L.orc_gen_grads.argtypes = [U64, U32, U32, U32, I32, I64, P]
        L.orc_moments_and_update.argtypes = [I64, P, P, P, P, D, D, D, D, I32, I64, P]
        L.orc_sumsq.argtypes = [I64, P]
        L.orc_sumsq.restype = D
        L.orc_trust_ratio.argtypes = [D, D, I32]
        L.orc_trust_ratio.restype = D
        L.orc_apply.argtypes = [I64, P, P, D, D]
        L.orc_lamb_tensor_step.argtypes = [I64, P, P, P, P, P, D, D, D, D, D, I32, I32, I64, P]
        L.orc_reduce.argtypes = [I64, I32, P, D, P]
        L.orc_bf16_neighbors.argtypes = [I64, P, P, P]
        L.orc_bf16_rne.argtypes = [D]
        L.orc_bf16_rne.restype = ctypes.c_uint16
        L.orc_num_threads.restype = I32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def f32(x: float) -> float:
    """The fp32 value of a hyper-parameter, promoted exactly to double (reading Z6)."""
    return float(np.float32(x))


# ---------------------------------------------------------------- generator
def philox4x32_10(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return list(o)


def rank_term(mode: int, rank: int) -> int:
    return 0 if mode == REPLICATED else rank + 1


def gen_weights(seed: int, tensor_id: int, init: int, numel: int) -> np.ndarray:
    out = np.empty(numel, np.float64)
    lib().orc_gen_weights(seed, tensor_id, init, numel, _p(out))
    return out


def gen_grads(seed: int, rterm: int, tensor_id: int, step: int, gexp: int, numel: int) -> np.ndarray:
    out = np.empty(numel, np.float64)
    lib().orc_gen_grads(seed, rterm, tensor_id, step, gexp, numel, _p(out))
    return out


def reduce(G: List[np.ndarray], grad_scale: float) -> np.ndarray:
    n = G[0].size
    arr = (ctypes.c_void_p * len(G))(*[_p(g).value for g in G])
    out = np.empty(n, np.float64)
    lib().orc_reduce(n, len(G), arr, grad_scale, _p(out))
    return out


def bf16_neighbors(x: np.ndarray):
    """(lo, hi): the bf16 numbers bracketing each x (equal where x is a bf16 number) — the two
    values the NVSwitch's reduction may return for an exact sum x (reading Z23)."""
    x = np.ascontiguousarray(x, np.float64)
    lo, hi = np.empty_like(x), np.empty_like(x)
    lib().orc_bf16_neighbors(x.size, _p(x), _p(lo), _p(hi))
    return lo, hi


def bf16_rne_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns of RNE(float32(x)) — vectorised restatement checked against
    orc_bf16_rne in tests."""
    f = np.asarray(x, np.float64).astype(np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) >> 16).astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        r[nan] = ((b[nan] >> 16) | 0x40).astype(np.uint16)
    return r


# ---------------------------------------------------------------- LAMB, one tensor
def lamb_tensor_step(w: np.ndarray, m: np.ndarray, v: np.ndarray, g: np.ndarray, group, t: int):
    """In-place LAMB step of one tensor in double.  `group` has lr, beta1, beta2, eps,
    weight_decay, adapt, bias_correction; their fp32 values are promoted (Z6).
    Returns (||w||, ||u||, ratio)."""
    n = w.size
    u = np.empty(n, np.float64)
    out3 = np.empty(3, np.float64)
    lib().orc_lamb_tensor_step(n, _p(w), _p(m), _p(v), _p(np.ascontiguousarray(g, np.float64)), _p(u),
                               f32(group.lr), f32(group.beta1), f32(group.beta2), f32(group.eps),
                               f32(group.weight_decay), int(group.adapt), int(group.bias_correction),
                               int(t), _p(out3))
    return float(out3[0]), float(out3[1]), float(out3[2])


def moments_and_update(w, m, v, g, group, t) -> np.ndarray:
    u = np.empty(w.size, np.float64)
    lib().orc_moments_and_update(w.size, _p(w), _p(m), _p(v), _p(np.ascontiguousarray(g, np.float64)),
                                 f32(group.beta1), f32(group.beta2), f32(group.eps),
                                 f32(group.weight_decay), int(group.bias_correction), int(t), _p(u))
    return u


def sumsq(x: np.ndarray) -> float:
    return lib().orc_sumsq(x.size, _p(np.ascontiguousarray(x, np.float64)))


def trust_ratio(w_norm: float, u_norm: float, adapt: int) -> float:
    return lib().orc_trust_ratio(w_norm, u_norm, adapt)


def apply(w: np.ndarray, u: np.ndarray, lr: float, ratio: float) -> None:
    lib().orc_apply(w.size, _p(w), _p(u), lr, ratio)


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ---------------------------------------------------------------- whole workload
class OracleRun:
    """Unsharded LAMB over (a subset of) a workload's tensors, state in double.

    Gradients come from the generator per rank j < world_size and are reduced with
    grad_scale (default 1/D).  Every tensor's result depends only on its own data, so
    a subset gives the exact oracle values of those tensors at any size.
    """

    def __init__(self, workload, world_size: int = 1, mode: int = PER_RANK,
                 tensor_ids: Optional[Iterable[int]] = None, grad_scale: Optional[float] = None,
                 groups=None):
        self.wl = workload
        self.D = world_size
        self.mode = mode
        self.groups = groups if groups is not None else workload.groups
        self.grad_scale = (1.0 / world_size) if grad_scale is None else grad_scale
        self.ids = list(range(len(workload.tensors))) if tensor_ids is None else list(tensor_ids)
        self.w: Dict[int, np.ndarray] = {}
        self.m: Dict[int, np.ndarray] = {}
        self.v: Dict[int, np.ndarray] = {}
        self.stats: Dict[int, tuple] = {}
        # w before the most recent step (tests compare the per-step update dw = w - w_prev)
        self.w_prev: Dict[int, np.ndarray] = {}
        for i in self.ids:
            ts = workload.tensors[i]
            self.w[i] = gen_weights(workload.seed, i, ts.init, ts.numel)
            self.m[i] = np.zeros(ts.numel)
            self.v[i] = np.zeros(ts.numel)

    def grads(self, i: int, step: int) -> np.ndarray:
        ts = self.wl.tensors[i]
        ranks = [0] if self.mode == REPLICATED else list(range(self.D))
        G = [gen_grads(self.wl.seed, rank_term(self.mode, j), i, step, ts.gexp, ts.numel) for j in ranks]
        if self.mode == REPLICATED:
            G = G * self.D
        return reduce(G, f32(self.grad_scale))

    def step(self, t: int, max_grad_norm: float = 0.0, inv_loss_scale: float = 1.0) -> dict:
        """One LAMB step.  With the pre-step of SURVEY §8(f) NEXT #3 (reading Z12'):
        g <- g * inv_loss_scale; gn = ||g|| over ALL tensors of the workload; skip the step
        (state untouched) if gn is not finite; if max_grad_norm > 0 and
        c = max_grad_norm / (gn + 1e-6) < 1, g <- c * g (torch clip_grad_norm_ rule)."""
        info = {"grad_norm": None, "clip": 1.0, "skipped": False}
        for i in self.ids:
            self.w_prev[i] = self.w[i].copy()
        if max_grad_norm > 0.0 or inv_loss_scale != 1.0:
            gsq = 0.0
            for i in range(len(self.wl.tensors)):          # the GLOBAL norm needs every tensor
                gsq += sumsq(self.grads(i, t) * f32(inv_loss_scale))
            gn = float(np.sqrt(gsq))
            info["grad_norm"] = gn
            if not np.isfinite(gn):
                info["skipped"] = True
                return info
            if max_grad_norm > 0.0:
                c = f32(max_grad_norm) / (gn + 1e-6)
                info["clip"] = min(1.0, c)
        scale = f32(inv_loss_scale) * info["clip"]
        for i in self.ids:
            g = self.grads(i, t)
            if scale != 1.0:
                g = g * scale
            grp = self.groups[self.wl.tensors[i].group]
            self.stats[i] = lamb_tensor_step(self.w[i], self.m[i], self.v[i], g, grp, t)
        return info


def sharded_step(wl, pl: OraclePlan, w_flat: np.ndarray, m_flat: np.ndarray, v_flat: np.ndarray,
                 g_flat: np.ndarray, t: int, groups=None) -> Dict[int, tuple]:
    """Brute-force ZeRO-2 style step over the plan's shards (H8): every rank updates its
    own segments, partial ||w||^2 / ||u||^2 are combined over ranks in order r = 0..D-1,
    and the ratio is applied per segment.  Arrays are flat (plan layout) doubles; updated
    in place.  Returns per-tensor (||w||, ||u||, ratio)."""
    groups = groups if groups is not None else wl.groups
    T = len(wl.tensors)
    W2 = [0.0] * T
    U2 = [0.0] * T
    us = []  # per rank, per segment u
    for r in range(pl.world_size):
        us_r = []
        for (i, shard_off, toff, ln) in pl.segments[r]:
            f = pl.tensor_off[i] + toff
            sl = slice(f, f + ln)
            grp = groups[wl.tensors[i].group]
            w_seg = np.ascontiguousarray(w_flat[sl])
            m_seg = np.ascontiguousarray(m_flat[sl])
            v_seg = np.ascontiguousarray(v_flat[sl])
            u = moments_and_update(w_seg, m_seg, v_seg, g_flat[sl], grp, t)
            m_flat[sl] = m_seg
            v_flat[sl] = v_seg
            us_r.append(u)
        us.append(us_r)
    for r in range(pl.world_size):   # fixed combine order
        for k, (i, shard_off, toff, ln) in enumerate(pl.segments[r]):
            f = pl.tensor_off[i] + toff
            W2[i] += sumsq(w_flat[f:f + ln])
            U2[i] += sumsq(us[r][k])
    stats = {}
    for i in range(T):
        grp = groups[wl.tensors[i].group]
        wn, un = float(np.sqrt(W2[i])), float(np.sqrt(U2[i]))
        stats[i] = (wn, un, trust_ratio(wn, un, grp.adapt))
    for r in range(pl.world_size):
        for k, (i, shard_off, toff, ln) in enumerate(pl.segments[r]):
            f = pl.tensor_off[i] + toff
            seg = np.ascontiguousarray(w_flat[f:f + ln])
            apply(seg, us[r][k], f32(groups[wl.tensors[i].group].lr), stats[i][2])
            w_flat[f:f + ln] = seg
    return stats
