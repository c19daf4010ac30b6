"""`LambOptimizer`: use the sharded LAMB step from a PyTorch training loop.

Marshalling only — the step is `lamb_step` of liblamb.so.  The model's parameters are re-pointed
to views of the library's flat bf16 PARAM buffer, and their `.grad` to views of the flat bf16
GRAD buffer, so autograd accumulates straight into the buffer the fused reduce-scatter reads
and the updated (all-gathered) bf16 parameters are what the next forward uses — no copies.
The fp32 master weights and Adam moments live in the library's shards (ZeRO-2, §2
P:689-701); LAMB per PAPER.md §3.1 P:288-293 (update rule and readings: DESIGN.md §3).

    opt = LambOptimizer(model.parameters(), lr=1e-3, weight_decay=0.01, pg=dist.group.WORLD)
    for batch in data:
        opt.zero_grad()
        loss(model(batch)).backward()
        opt.step()

Parameter groups follow torch.optim conventions ([{"params": [...], "lr": ..., ...}, ...]).
Parameters must be bf16 CUDA tensors on this rank's device.

`overlap=True` (D > 1) runs the paper's DP overlap (§3.2) on the copy engines
(DESIGN.md §7b #2b): a post-accumulate-grad hook pushes each bucket's gradients to the peers'
staging as soon as the backward has produced all of them (`lamb_push_grads_bucket`), `step()`
runs `lamb_step_staged` (the all-gather then streams into the next forward), and a global
module forward-pre-hook makes the forward of a module wait for the buckets its own parameters
live in (`lamb_wait_params_bucket`).  Parameters must therefore be used through `nn.Module`
forwards; results are bit-identical to `overlap=False`.  Gradient accumulation: run every
micro-batch but the last under `with opt.no_sync():` (as with DDP) — the buckets are pushed by
the last backward only, once their gradients are final.  A second backward outside `no_sync()`
before `step()` raises instead of reducing a partial gradient.
"""
from __future__ import annotations

import contextlib
from typing import Iterable, List, Optional

import torch

from . import lamb


class LambOptimizer:
    def __init__(self, params: Iterable, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-6,
                 weight_decay: float = 0.0, adapt: bool = True, bias_correction: bool = True,
                 world_size: int = 1, rank: int = 0, pg=None, comm_mode: int = lamb.LAMB_COMM_FUSED,
                 bucket_cap: int = 0, max_grad_norm: float = 0.0, graph: bool = False,
                 overlap: bool = False, bootstrap: str = "nccl"):
        params = list(params)
        if params and not isinstance(params[0], dict):
            params = [{"params": params}]
        defaults = dict(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay,
                        adapt=int(adapt), bias_correction=int(bias_correction))
        self.groups: List[dict] = []
        self.params: List[torch.nn.Parameter] = []
        table = []
        for gi, g in enumerate(params):
            hp = dict(defaults)
            for k_in, k_out in (("lr", "lr"), ("eps", "eps"), ("weight_decay", "weight_decay")):
                if k_in in g:
                    hp[k_out] = g[k_in]
            if "betas" in g:
                hp["beta1"], hp["beta2"] = g["betas"]
            self.groups.append(hp)
            for p in g["params"]:
                if p.dtype != torch.bfloat16 or not p.is_cuda:
                    raise TypeError("LambOptimizer manages bf16 CUDA parameters")
                self.params.append(p)
                table.append((p.numel(), gi))
        if not self.params:
            raise ValueError("no parameters")
        self.device = self.params[0].device.index or 0
        self.overlap = bool(overlap) and world_size > 1
        if self.overlap and (comm_mode != lamb.LAMB_COMM_FUSED or max_grad_norm > 0):
            raise ValueError("overlap=True needs comm_mode=FUSED and no global clipping")
        self.L = lamb.Lamb(table, self.groups, world_size=world_size, rank=rank, device=self.device,
                           comm_mode=comm_mode, bucket_cap=bucket_cap, pg=pg, graph=graph, ce=self.overlap,
                           bootstrap=bootstrap)
        # fp32 master = the current bf16 values (exact), then the params become buffer views
        flat = torch.zeros(self.L.plan.flat_size, dtype=torch.float32, device=f"cuda:{self.device}")
        for p, off in zip(self.params, self.L.plan.tensor_off.tolist()):
            flat[off:off + p.numel()] = p.detach().reshape(-1).float()
        self.L.set_master(flat)
        del flat
        pv, gv = self.L.param_views(), self.L.grad_views()
        for p, v, g in zip(self.params, pv, gv):
            p.data = v.view(p.shape)
            p.grad = g.view(p.shape)
        self._gviews = [p.grad for p in self.params]   # cached: step() compares pointers only
        if max_grad_norm > 0:
            self.L.set_grad_clip(max_grad_norm)
        self.t = 0
        self._hooks = []
        if self.overlap:
            self._setup_overlap()

    # ---------------- copy-engine overlap (overlap=True)
    def _setup_overlap(self) -> None:
        self._ov = BucketOverlap(self.params, self.L.plan.tensor_bucket.tolist(), int(self.L.plan.buckets.shape[0]),
                                 push=self.L.push_grads_bucket, wait=self.L.wait_params_bucket,
                                 grad_views=[g.view(p.shape) for p, g in zip(self.params, self.L.grad_views())])
        self._hooks = self._ov.install()

    @contextlib.contextmanager
    def no_sync(self):
        """Backward passes inside this context only accumulate into the grad buffer (gradient
        accumulation micro-batches); with overlap=True they push nothing to the peers.  The
        backward of the last micro-batch runs outside it.  With overlap=False a no-op."""
        if not self.overlap:
            yield
            return
        prev = self._ov.sync
        self._ov.sync = False
        try:
            yield
        finally:
            self._ov.sync = prev

    def wait_params(self) -> None:
        """Make the current stream wait for every bucket's all-gather (e.g. before using the
        parameters outside a module forward)."""
        if self.overlap:
            self._ov.wait_all()

    def close(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []
        self.L.close()

    @torch.no_grad()
    def zero_grad(self, set_to_none: bool = False) -> None:
        # the grad views ARE the library's flat buffer (padding stays zero)
        self.L.grad_buffer().zero_()

    @torch.no_grad()
    def step(self, closure=None) -> None:
        if self.overlap:
            self._ov.before_step(self.t + 1)   # pending waits and pushes of this step
            self.t += 1
            self.L.step_staged(self.t)
            self._ov.after_step(self.t)
            return
        for p, g in zip(self.params, self._gviews):   # autograd may have replaced .grad
            if p.grad is not None and p.grad.data_ptr() != g.data_ptr():
                g.copy_(p.grad)
                p.grad = g
        self.t += 1
        self.L.step(self.t)

    def set_lr(self, lr: float, group: Optional[int] = None) -> None:
        for gi in ([group] if group is not None else range(len(self.groups))):
            self.L.set_lr(gi, lr)

    def state_dict_path(self, path: str) -> None:
        """Two-stage checkpoint of the sharded state (lamb_checkpoint_save)."""
        self.L.checkpoint_save(path, self.t)

    def load_path(self, path: str) -> None:
        self.t = self.L.checkpoint_load(path)
        if self.overlap:   # the load rebuilt every param buffer: nothing to wait for or push
            self._ov.reset(self.t)


class BucketOverlap:
    """Host bookkeeping of the copy-engine overlap (pure Python; the GPU work is in `push` /
    `wait`).  Per training step: `push(b, t)` exactly once per bucket, as soon as the backward
    has accumulated the gradient of the bucket's last parameter (post-accumulate-grad hooks);
    per forward after a staged step: `wait(b, t_staged)` once per bucket, right before the first
    module whose own parameters live in bucket b runs (a global module forward-pre-hook).
    `before_step` pushes buckets whose parameters got no gradient and waits for buckets no
    module used; `after_step` arms the next forward's waits.  While `sync` is False (the
    optimizer's no_sync(): accumulation micro-batches) the hooks push nothing; a bucket whose
    parameters receive gradients again after it was pushed raises (its pushed copy would be
    partial, and the copy engine may still be reading the buffer the backward writes)."""

    def __init__(self, params, bucket_of, n_buckets: int, push, wait, grad_views=None):
        self.params = list(params)
        self.n = n_buckets
        self.push, self.wait = push, wait
        self.grad_views = grad_views
        self.size = [0] * n_buckets
        self.bucket_of = {}
        for p, b in zip(self.params, bucket_of):
            self.size[b] += 1
            self.bucket_of[id(p)] = b
        self.pending = list(self.size)
        self.pushed = [False] * n_buckets
        self.staged = 0
        self.awaited = [True] * n_buckets
        self.t_next = 1
        self.sync = True

    def install(self):
        hooks = []
        for i, p in enumerate(self.params):
            hooks.append(p.register_post_accumulate_grad_hook(self._grad_hook(i)))
        hooks.append(torch.nn.modules.module.register_module_forward_pre_hook(self._pre_hook))
        return hooks

    def _grad_hook(self, i):
        b = self.bucket_of[id(self.params[i])]
        gview = self.grad_views[i] if self.grad_views is not None else None

        def hook(param):
            if gview is not None and param.grad is not None and param.grad.data_ptr() != gview.data_ptr():
                gview.copy_(param.grad)   # autograd replaced .grad: back into the library buffer
                param.grad = gview
            if not self.sync:
                return
            if self.pushed[b]:
                raise RuntimeError(
                    f"bucket {b} received gradients after it was pushed to the peers in this step: "
                    "with LambOptimizer(overlap=True) run the backward of every micro-batch but the "
                    "last under `with opt.no_sync():`")
            self.pending[b] -= 1
            if self.pending[b] == 0 and not self.pushed[b]:
                self.push(b, self.t_next)
                self.pushed[b] = True
        return hook

    def _pre_hook(self, module, args):
        if not self.staged:
            return
        for p in module.parameters(recurse=False):
            b = self.bucket_of.get(id(p))
            if b is not None and not self.awaited[b]:
                self.wait(b, self.staged)
                self.awaited[b] = True

    def wait_all(self):
        if self.staged:
            for b in range(self.n):
                if not self.awaited[b]:
                    self.wait(b, self.staged)
                    self.awaited[b] = True

    def before_step(self, t: int):
        self.wait_all()   # (a forward that skipped some modules)
        for b in range(self.n):   # buckets whose params got no gradient this step
            if not self.pushed[b]:
                self.push(b, t)
                self.pushed[b] = True

    def reset(self, t: int):
        """After a checkpoint load at step t: no pending waits, the next pushes are step t+1."""
        self.staged = 0
        self.t_next = t + 1
        self.pending = list(self.size)
        self.pushed = [False] * self.n
        self.awaited = [True] * self.n

    def after_step(self, t: int):
        self.staged = t
        self.t_next = t + 1
        self.pending = list(self.size)
        self.pushed = [False] * self.n
        self.awaited = [False] * self.n
