"""Thin Python binding of liblamb.so (include/lamb.h, include/lamb_synth.h).

Argument marshalling only: every step of the LAMB path runs in the library's CUDA kernels.
PyTorch is used for device memory views, streams and the process group (unique-id
broadcast).  There is no fallback: if liblamb.so is missing this module raises on import.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LAMB_DEBUG_LIB=1 loads the -DLAMB_DEBUG build (device-side bounds / ring-tag / bounded-wait
# checks standing in for compute-sanitizer): same kernels and arithmetic, so the
# results are the same; a failed check prints "LAMB_DEBUG ..." and traps
DEBUG = os.environ.get("LAMB_DEBUG_LIB", "0") not in ("", "0")
LIB_PATH = os.path.join(_HERE, "liblamb_debug.so" if DEBUG else "liblamb.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2402_15627_b200.build` "
                      "(there is no CPU fallback)")
_L = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
LAMB_OK, LAMB_EINVAL, LAMB_ENOMEM, LAMB_ECUDA, LAMB_ENCCL, LAMB_ESTATE, LAMB_EUNSUPPORTED = range(7)
STATUS_NAMES = ["LAMB_OK", "LAMB_EINVAL", "LAMB_ENOMEM", "LAMB_ECUDA", "LAMB_ENCCL", "LAMB_ESTATE",
                "LAMB_EUNSUPPORTED"]
LAMB_MAX_GROUPS = 64
LAMB_MAX_RANKS = 8
LAMB_UNIQUE_ID_BYTES = 128
LAMB_COMM_NCCL, LAMB_COMM_FUSED, LAMB_COMM_NVLS = 0, 1, 2
LAMB_FLAG_TIMING = 1
LAMB_FLAG_GRAPH = 2
LAMB_FLAG_CE = 4
LAMB_BUCKET_DEFER_AG = 1
LAMB_BUF_GRAD, LAMB_BUF_PARAM, LAMB_BUF_W, LAMB_BUF_M, LAMB_BUF_V, LAMB_BUF_GSUM = range(6)
PHASES = ["barrier_in", "pass_a", "finalize", "exchange", "pass_b", "barrier_out"]
LAMB_N_PHASES = len(PHASES)


# ---------------------------------------------------------------- structs
class lamb_tensor(ctypes.Structure):
    _fields_ = [("numel", ctypes.c_int64), ("group", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class lamb_group(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("adapt", ctypes.c_int32), ("bias_correction", ctypes.c_int32)]


class lamb_config(ctypes.Structure):
    _fields_ = [("world_size", ctypes.c_int32), ("rank", ctypes.c_int32), ("device", ctypes.c_int32),
                ("comm_mode", ctypes.c_int32), ("bucket_cap_elems", ctypes.c_int64),
                ("grad_scale", ctypes.c_float), ("flags", ctypes.c_int32)]


_P64 = ctypes.POINTER(ctypes.c_int64)


class lamb_plan_view(ctypes.Structure):
    _fields_ = [("n_tensors", ctypes.c_int64), ("n_buckets", ctypes.c_int64),
                ("n_segments", ctypes.c_int64), ("n_straddlers", ctypes.c_int64),
                ("flat_size", ctypes.c_int64), ("shard_size", ctypes.c_int64),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("tensor_off", _P64), ("tensor_bucket", _P64), ("buckets", _P64),
                ("segments", _P64), ("straddlers", _P64)]


class lamb_step_info(ctypes.Structure):
    _fields_ = [("grad_norm", ctypes.c_double), ("clip", ctypes.c_float), ("skipped", ctypes.c_int32)]


class lamb_synth_tensor(ctypes.Structure):
    _fields_ = [("init", ctypes.c_int32), ("gexp", ctypes.c_int32)]


# ---------------------------------------------------------------- signatures
_st = ctypes.c_int
_vp = ctypes.c_void_p
_SIGS = {
    "lamb_plan_create": (_st, [ctypes.POINTER(lamb_tensor), ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                               ctypes.c_int64, ctypes.POINTER(_vp)]),
    "lamb_plan_get": (_st, [_vp, ctypes.POINTER(lamb_plan_view)]),
    "lamb_plan_destroy": (None, [_vp]),
    "lamb_get_unique_id": (_st, [ctypes.c_char_p]),
    "lamb_create": (_st, [ctypes.POINTER(lamb_tensor), ctypes.c_int64, ctypes.POINTER(lamb_group),
                          ctypes.c_int32, ctypes.POINTER(lamb_config), ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "lamb_create_with_allgather": (_st, [ctypes.POINTER(lamb_tensor), ctypes.c_int64, ctypes.POINTER(lamb_group),
                                         ctypes.c_int32, ctypes.POINTER(lamb_config), _vp, _vp,
                                         ctypes.POINTER(_vp)]),
    "lamb_step": (_st, [_vp, _vp, ctypes.c_int64, _vp]),
    "lamb_step_host": (_st, [_vp, _vp, _vp, ctypes.c_int64, _vp]),
    "lamb_step_bucket": (_st, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _vp]),
    "lamb_gather_bucket": (_st, [_vp, ctypes.c_int64, _vp]),
    "lamb_push_grads_bucket": (_st, [_vp, ctypes.c_int64, ctypes.c_int64, _vp]),
    "lamb_step_staged": (_st, [_vp, ctypes.c_int64, _vp]),
    "lamb_wait_params_bucket": (_st, [_vp, ctypes.c_int64, ctypes.c_int64, _vp]),
    "lamb_set_max_ctas": (_st, [_vp, ctypes.c_int32]),
    "lamb_self_check": (_st, [_vp, _vp, _vp]),
    "lamb_sm_partition": (_st, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                ctypes.POINTER(ctypes.c_int32)]),
    "lamb_destroy": (None, [_vp]),
    "lamb_query_plan": (_st, [_vp, ctypes.POINTER(lamb_plan_view)]),
    "lamb_buffer": (_st, [_vp, ctypes.c_int32, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64)]),
    "lamb_set_master": (_st, [_vp, _vp, ctypes.c_int32, _vp]),
    "lamb_get_state": (_st, [_vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp]),
    "lamb_get_tensor_stats": (_st, [_vp, _vp, _vp, _vp]),
    "lamb_set_lr": (_st, [_vp, ctypes.c_int32, ctypes.c_float]),
    "lamb_set_grad_clip": (_st, [_vp, ctypes.c_float]),
    "lamb_set_loss_scale": (_st, [_vp, ctypes.c_float]),
    "lamb_get_step_info": (_st, [_vp, ctypes.POINTER(lamb_step_info)]),
    "lamb_checkpoint_save": (_st, [_vp, ctypes.c_char_p, ctypes.c_int64, _vp]),
    "lamb_checkpoint_wait": (_st, [_vp]),
    "lamb_checkpoint_load": (_st, [_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), _vp]),
    "lamb_timing_begin": (_st, [_vp, ctypes.c_int32]),
    "lamb_timing_read": (_st, [_vp, _vp, ctypes.POINTER(ctypes.c_int32)]),
    "lamb_launch_count": (ctypes.c_int64, [_vp]),
    "lamb_last_error": (ctypes.c_char_p, [_vp]),
    "lamb_synth_init": (_st, [_vp, ctypes.POINTER(lamb_synth_tensor), ctypes.c_uint64, _vp]),
    "lamb_synth_grads": (_st, [_vp, ctypes.POINTER(lamb_synth_tensor), ctypes.c_uint64, ctypes.c_uint32,
                               ctypes.c_uint32, _vp]),
    "lamb_synth_philox": (_st, [_vp, _vp, _vp]),
}
if DEBUG:
    _SIGS["lamb_debug_corrupt_item"] = (_st, [_vp, ctypes.c_int64, ctypes.c_int64])
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_L, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


class LambError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


def check(status: int, handle=None) -> None:
    if status != LAMB_OK:
        raise LambError(status, (lamb_last_error(handle) or b"").decode())


def exported_symbols() -> List[str]:
    return list(_SIGS)


# ---------------------------------------------------------------- plan
class PlanView:
    """Host copy of a lamb_plan_view (numpy int64 tables)."""

    def __init__(self, v: lamb_plan_view):
        def arr(p, n, k=1):
            if n == 0:
                return np.zeros((0, k) if k > 1 else 0, np.int64)
            a = np.ctypeslib.as_array(p, shape=(n * k,)).copy()
            return a.reshape(n, k) if k > 1 else a
        self.n_tensors, self.flat_size, self.shard_size = v.n_tensors, v.flat_size, v.shard_size
        self.world_size, self.rank = v.world_size, v.rank
        self.tensor_off = arr(v.tensor_off, v.n_tensors)
        self.tensor_bucket = arr(v.tensor_bucket, v.n_tensors)
        self.buckets = arr(v.buckets, v.n_buckets, 4)
        self.segments = arr(v.segments, v.n_segments, 4)
        self.straddlers = arr(v.straddlers, v.n_straddlers)


def _tensor_array(numels: Sequence[int], groups: Sequence[int]):
    arr = (lamb_tensor * len(numels))()
    for i, (n, g) in enumerate(zip(numels, groups)):
        arr[i].numel, arr[i].group, arr[i].reserved = int(n), int(g), 0
    return arr


def host_plan(numels: Sequence[int], world_size: int, rank: int, cap: int = 0,
              groups: Optional[Sequence[int]] = None) -> PlanView:
    """The library's planner (row a0) on the host; no GPU needed."""
    groups = groups if groups is not None else [0] * len(numels)
    arr = _tensor_array(numels, groups)
    h = _vp()
    check(lamb_plan_create(arr, len(numels), world_size, rank, cap, ctypes.byref(h)))
    try:
        v = lamb_plan_view()
        check(lamb_plan_get(h, ctypes.byref(v)))
        return PlanView(v)
    finally:
        lamb_plan_destroy(h)


def device_philox(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    check(lamb_synth_philox(c, k, o))
    return list(o)


def sm_partition(device: int, lamb_sms: int):
    """(lamb_stream_ptr, compute_stream_ptr, sms) — two green-context streams (see lamb.h)."""
    a, b, n = _vp(), _vp(), ctypes.c_int32()
    check(lamb_sm_partition(device, lamb_sms, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
    return a.value, b.value, n.value


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(LAMB_UNIQUE_ID_BYTES)
    check(lamb_get_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------- handle
class Lamb:
    """One sharded LAMB optimizer instance (one per rank).

    tensors: list of (numel, group); groups: list of objects/dicts with lr, beta1, beta2,
    eps, weight_decay, adapt, bias_correction.  For world_size > 1 pass `unique_id`
    (rank 0's get_unique_id(), broadcast by the caller) or a torch process group `pg`.
    """

    def __init__(self, tensors: Sequence[tuple], groups: Sequence, world_size: int = 1, rank: int = 0,
                 device: int = 0, comm_mode: int = LAMB_COMM_FUSED, bucket_cap: int = 0,
                 grad_scale: float = 0.0, timing: bool = False, unique_id: Optional[bytes] = None,
                 pg=None, graph: bool = False, bootstrap: str = "nccl", ce: bool = False):
        import torch
        self.torch = torch
        self.device = device
        numels = [int(t[0]) for t in tensors]
        grp = [int(t[1]) for t in tensors]
        self._tensors = _tensor_array(numels, grp)
        self.n_tensors = len(numels)
        self.numels = numels
        garr = (lamb_group * len(groups))()
        for k, g in enumerate(groups):
            get = (lambda name: g[name]) if isinstance(g, dict) else (lambda name: getattr(g, name))
            garr[k].lr, garr[k].beta1, garr[k].beta2 = get("lr"), get("beta1"), get("beta2")
            garr[k].eps, garr[k].weight_decay = get("eps"), get("weight_decay")
            garr[k].adapt, garr[k].bias_correction = int(get("adapt")), int(get("bias_correction"))
        cfg = lamb_config(world_size, rank, device, comm_mode, bucket_cap, grad_scale,
                          (LAMB_FLAG_TIMING if timing else 0) | (LAMB_FLAG_GRAPH if graph else 0) |
                          (LAMB_FLAG_CE if ce else 0))
        self.h = _vp()
        if world_size > 1 and bootstrap == "host":
            # FUSED / NVLS without an NCCL communicator: handles exchanged over the caller's group
            if pg is None:
                raise ValueError("bootstrap='host' needs a process group")
            ag = _pg_allgather(pg)
            _ag_errors.clear()
            st = lamb_create_with_allgather(self._tensors, len(numels), garr, len(groups), ctypes.byref(cfg),
                                            ctypes.cast(ag, _vp), None, ctypes.byref(self.h))
            if st != LAMB_OK:
                msg = (lamb_last_error(None) or b"").decode()
                raise LambError(st, msg + (" (" + "; ".join(_ag_errors) + ")" if _ag_errors else ""))
        else:
            if bootstrap != "nccl":
                raise ValueError("bootstrap must be 'nccl' or 'host'")
            if world_size > 1 and unique_id is None:
                if pg is None:
                    raise ValueError("world_size > 1 needs unique_id or a process group")
                unique_id = broadcast_unique_id(pg, rank, device)
            check(lamb_create(self._tensors, len(numels), garr, len(groups), ctypes.byref(cfg),
                              unique_id, ctypes.byref(self.h)))
        v = lamb_plan_view()
        check(lamb_query_plan(self.h, ctypes.byref(v)), self.h)
        self.plan = PlanView(v)
        self.world_size, self.rank = world_size, rank

    # -- buffers as torch views (no copies)
    def _buf(self, which: int, dtype):
        torch = self.torch
        ptr, n = _vp(), ctypes.c_int64()
        check(lamb_buffer(self.h, which, ctypes.byref(ptr), ctypes.byref(n)), self.h)
        return _torch_view(ptr.value, n.value, dtype, self.device)

    def grad_buffer(self):
        return self._buf(LAMB_BUF_GRAD, self.torch.bfloat16)

    def param_buffer(self):
        return self._buf(LAMB_BUF_PARAM, self.torch.bfloat16)

    def state_buffer(self, which: int):
        return self._buf(which, self.torch.float32)

    def grad_views(self):
        g = self.grad_buffer()
        return [g[o:o + n] for o, n in zip(self.plan.tensor_off, self.numels)]

    def param_views(self):
        p = self.param_buffer()
        return [p[o:o + n] for o, n in zip(self.plan.tensor_off, self.numels)]

    # -- the step
    def _stream(self, stream):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def step(self, t: int, stream=None, grads_ptr: Optional[int] = None) -> None:
        check(lamb_step(self.h, grads_ptr, int(t), self._stream(stream)), self.h)

    def step_bucket(self, bucket: int, t: int, defer_ag: bool = False, stream=None) -> None:
        check(lamb_step_bucket(self.h, int(bucket), int(t), LAMB_BUCKET_DEFER_AG if defer_ag else 0,
                               self._stream(stream)), self.h)

    def self_check(self) -> dict:
        """lamb_self_check: device-side audit (§4.3); all counts zero = healthy."""
        c = (ctypes.c_int64 * 5)()
        check(lamb_self_check(self.h, c, self._stream(None)), self.h)
        keys = ("nonfinite_state", "param_mismatch", "shard_padding_nonzero", "flat_padding_nonzero",
                "peer_unreachable")
        return dict(zip(keys, list(c)))

    def set_max_ctas(self, max_ctas: int) -> None:
        check(lamb_set_max_ctas(self.h, int(max_ctas)), self.h)

    def gather_bucket(self, bucket: int, stream=None) -> None:
        check(lamb_gather_bucket(self.h, int(bucket), self._stream(stream)), self.h)

    # copy-engine schedule (ce=True at construction): RS pushes during the backward, the update
    # after it, the AG pushes into the next forward
    def push_grads_bucket(self, bucket: int, t: int, stream=None) -> None:
        check(lamb_push_grads_bucket(self.h, int(bucket), int(t), self._stream(stream)), self.h)

    def step_staged(self, t: int, stream=None) -> None:
        check(lamb_step_staged(self.h, int(t), self._stream(stream)), self.h)

    def wait_params_bucket(self, bucket: int, t: int, stream=None) -> None:
        check(lamb_wait_params_bucket(self.h, int(bucket), int(t), self._stream(stream)), self.h)

    def step_host(self, host_grads, host_params, t: int, stream=None) -> None:
        """host_grads / host_params: contiguous 2-byte CPU tensors (bf16 or int16 bit patterns)
        of flat_size elements, pinned for the copies to overlap."""
        n = self.plan.flat_size
        _check_flat(host_grads, n, _BF16_LIKE, "host_grads", cuda=False)
        _check_flat(host_params, n, _BF16_LIKE, "host_params", cuda=False)
        check(lamb_step_host(self.h, ctypes.c_void_p(host_grads.data_ptr()),
                             ctypes.c_void_p(host_params.data_ptr()), int(t), self._stream(stream)), self.h)

    # -- state
    def set_master(self, full_flat, stream=None) -> None:
        """full_flat: torch fp32 tensor (CPU or CUDA) of flat_size elements."""
        _check_flat(full_flat, self.plan.flat_size, ("torch.float32",), "full_flat",
                    cuda=None, device=self.device)
        on_dev = 1 if full_flat.is_cuda else 0
        check(lamb_set_master(self.h, ctypes.c_void_p(full_flat.data_ptr()), on_dev, self._stream(stream)), self.h)

    def synth_init(self, spec: Sequence[tuple], seed: int, stream=None) -> None:
        arr = (lamb_synth_tensor * len(spec))(*[lamb_synth_tensor(int(a), int(b)) for a, b in spec])
        check(lamb_synth_init(self.h, arr, seed, self._stream(stream)), self.h)

    def synth_grads(self, spec: Sequence[tuple], seed: int, rank_term: int, step: int, stream=None) -> None:
        arr = (lamb_synth_tensor * len(spec))(*[lamb_synth_tensor(int(a), int(b)) for a, b in spec])
        check(lamb_synth_grads(self.h, arr, seed, rank_term, step, self._stream(stream)), self.h)

    def get_state(self, which: int) -> np.ndarray:
        out = np.empty(self.plan.shard_size, np.float32)
        check(lamb_get_state(self.h, which, out.ctypes.data_as(_vp), 0, self._stream(None)), self.h)
        return out

    def tensor_stats(self):
        T = self.n_tensors
        w2, u2, r = np.empty(T), np.empty(T), np.empty(T, np.float32)
        check(lamb_get_tensor_stats(self.h, w2.ctypes.data_as(_vp), u2.ctypes.data_as(_vp),
                                    r.ctypes.data_as(_vp)), self.h)
        return w2, u2, r

    def set_lr(self, group: int, lr: float) -> None:
        check(lamb_set_lr(self.h, group, lr), self.h)

    # -- pre-step: clipping / loss scale / non-finite skip
    def set_grad_clip(self, max_grad_norm: float) -> None:
        check(lamb_set_grad_clip(self.h, max_grad_norm), self.h)

    def set_loss_scale(self, inv_loss_scale: float) -> None:
        check(lamb_set_loss_scale(self.h, inv_loss_scale), self.h)

    def step_info(self) -> dict:
        i = lamb_step_info()
        check(lamb_get_step_info(self.h, ctypes.byref(i)), self.h)
        return {"grad_norm": i.grad_norm, "clip": i.clip, "skipped": bool(i.skipped)}

    # -- checkpoint / resume (two-stage save, reshard on load)
    def checkpoint_save(self, path: str, step: int, stream=None) -> None:
        check(lamb_checkpoint_save(self.h, path.encode(), int(step), self._stream(stream)), self.h)

    def checkpoint_wait(self) -> None:
        check(lamb_checkpoint_wait(self.h), self.h)

    def checkpoint_load(self, path: str, stream=None) -> int:
        st = ctypes.c_int64()
        check(lamb_checkpoint_load(self.h, path.encode(), ctypes.byref(st), self._stream(stream)), self.h)
        return st.value

    def timing_begin(self, max_steps: int) -> None:
        check(lamb_timing_begin(self.h, max_steps), self.h)

    def timing_read(self) -> np.ndarray:
        n = ctypes.c_int32()
        check(lamb_timing_read(self.h, None, ctypes.byref(n)), self.h)
        out = np.zeros((n.value, LAMB_N_PHASES), np.float32)
        check(lamb_timing_read(self.h, out.ctypes.data_as(_vp), ctypes.byref(n)), self.h)
        return out

    def launch_count(self) -> int:
        return int(lamb_launch_count(self.h))

    def close(self) -> None:
        if getattr(self, "h", None) and self.h.value:
            lamb_destroy(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_BF16_LIKE = ("torch.bfloat16", "torch.int16", "torch.uint16")


def _check_flat(t, n: int, dtypes: Sequence[str], name: str, cuda: Optional[bool] = None,
                device: Optional[int] = None) -> None:
    """Validate a buffer handed to the library by pointer: the C side reads exactly n elements
    of the documented dtype from its first byte, so a wrong size, dtype, layout or device would
    be an out-of-bounds or garbage read, not an error."""
    if str(t.dtype) not in dtypes:
        raise ValueError(f"{name}: dtype {t.dtype}, expected one of {', '.join(dtypes)}")
    if t.numel() != n:
        raise ValueError(f"{name}: {t.numel()} elements, expected flat_size = {n}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if cuda is not None and bool(t.is_cuda) != cuda:
        raise ValueError(f"{name} must be a {'CUDA' if cuda else 'CPU'} tensor")
    if device is not None and t.is_cuda and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the handle on cuda:{device}")


_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


def _pg_allgather(pg):
    """lamb_allgather_fn over a torch.distributed group (bootstrap bytes only: IPC handles,
    the table hash).  The returned ctypes object must outlive the create call."""
    import torch.distributed as dist

    def fn(send, recv, nbytes, _user):
        try:
            out = [None] * dist.get_world_size(pg)
            dist.all_gather_object(out, ctypes.string_at(send, nbytes), group=pg)
            for j, b in enumerate(out):
                if len(b) != nbytes:
                    _ag_errors.append(f"rank {j} sent {len(b)} bootstrap bytes, expected {nbytes}")
                    return 1
                ctypes.memmove(recv + j * nbytes, b, nbytes)
            return 0
        except Exception as e:   # no exception may cross the C boundary: report it after the call
            _ag_errors.append(f"{type(e).__name__}: {e}")
            return 1
    return _ALLGATHER_FN(fn)


_ag_errors: List[str] = []   # messages of failed bootstrap all-gathers (appended to the LambError)


def broadcast_unique_id(pg, rank: int, device: int) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(pg)
    dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(LAMB_UNIQUE_ID_BYTES, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(get_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0, group=pg)
    return bytes(buf.cpu().numpy().tobytes())


def _torch_view(ptr: int, n: int, dtype, device: int):
    """A torch tensor aliasing library-owned device memory (valid until destroy)."""
    import torch
    itemsize = torch.empty(0, dtype=dtype).element_size()

    class _CAI:
        pass
    typestr = {torch.bfloat16: "<V2", torch.float32: "<f4"}[dtype]
    holder = _CAI()
    holder.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2" if dtype == torch.bfloat16 else typestr,
                                       "data": (ptr, False), "version": 3, "strides": None}
    with torch.cuda.device(device):
        t = torch.as_tensor(holder, device=f"cuda:{device}")
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    assert t.data_ptr() == ptr and t.numel() * itemsize == n * itemsize
    return t
