"""Pins of the oracle's pre-step: global grad-norm clipping, loss-scale
unscaling, non-finite skip — against torch.nn.utils.clip_grad_norm_ + torch.optim.AdamW
(float64), exact power-of-two loss scales, and the clipped-norm closed form."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from oracle import f32


def small_wl(adapt=1, seed=0):
    rng = np.random.default_rng(seed)
    ts = W.random_table(rng, 6, max_numel=500)
    groups = [W.GroupSpec(lr=1e-3, weight_decay=0.01, adapt=adapt), W.GroupSpec(lr=1e-3, adapt=adapt)]
    return W.Workload("clip", 80 + seed, ts, groups)


def test_huge_max_norm_is_identity():
    wl = small_wl()
    a, b = oracle.OracleRun(wl), oracle.OracleRun(wl)
    for t in (1, 2, 3):
        a.step(t)
        info = b.step(t, max_grad_norm=1e30)
        assert info["clip"] == 1.0 and info["grad_norm"] > 0
    for i in a.ids:
        assert np.array_equal(a.w[i], b.w[i]) and np.array_equal(a.m[i], b.m[i])


def test_power_of_two_loss_scale_is_exact():
    # grads scaled by S = 2^12 and unscaled by 1/S: bit-identical to unscaled training
    wl = small_wl()
    a, b = oracle.OracleRun(wl), oracle.OracleRun(wl)
    S = 2.0 ** 12
    orig = b.grads
    b.grads = lambda i, t: orig(i, t) * S
    for t in (1, 2):
        a.step(t)
        b.step(t, inv_loss_scale=1.0 / S)
    for i in a.ids:
        assert np.array_equal(a.w[i], b.w[i]) and np.array_equal(a.v[i], b.v[i])


@pytest.mark.parametrize("max_norm", [1e-3, 3e-2, 10.0])
def test_adapt0_clip_equals_torch_clip_grad_norm_and_adamw(max_norm):
    wl = small_wl(adapt=0, seed=3)
    orc = oracle.OracleRun(wl)
    params = [torch.tensor(orc.w[i].copy(), dtype=torch.float64, requires_grad=True) for i in orc.ids]
    pg = []
    for gi, grp in enumerate(wl.groups):
        ps = [p for i, p in zip(orc.ids, params) if wl.tensors[i].group == gi]
        pg.append({"params": ps, "lr": f32(grp.lr), "weight_decay": f32(grp.weight_decay)})
    opt = torch.optim.AdamW(pg, betas=(f32(0.9), f32(0.999)), eps=f32(1e-6))
    for t in range(1, 6):
        for i, p in zip(orc.ids, params):
            p.grad = torch.from_numpy(orc.grads(i, t))
        tn = torch.nn.utils.clip_grad_norm_(params, f32(max_norm))
        opt.step()
        info = orc.step(t, max_grad_norm=max_norm)
        assert info["grad_norm"] == pytest.approx(float(tn), rel=1e-13)
    for i, p in zip(orc.ids, params):
        assert np.max(np.abs(orc.w[i] - p.detach().numpy())) < 1e-13


def test_clipped_norm_closed_form_and_nonfinite_skip():
    wl = small_wl()
    orc = oracle.OracleRun(wl)
    g = {i: orc.grads(i, 1) for i in orc.ids}
    gn = np.sqrt(sum(np.sum(x * x) for x in g.values()))
    info = orc.step(1, max_grad_norm=gn / 4)
    assert info["clip"] == pytest.approx(f32(gn / 4) / (gn + 1e-6), rel=1e-15)
    assert info["clip"] * gn == pytest.approx(f32(gn / 4), rel=1e-4)
    # one non-finite gradient anywhere skips the whole step
    orc2 = oracle.OracleRun(wl)
    w0 = {i: orc2.w[i].copy() for i in orc2.ids}
    orig = orc2.grads
    orc2.grads = lambda i, t: (lambda x: (x.__setitem__(0, np.inf) or x) if i == 2 else x)(orig(i, t))
    info = orc2.step(1, max_grad_norm=1.0)
    assert info["skipped"] and all(np.array_equal(w0[i], orc2.w[i]) for i in orc2.ids)
    assert all(not orc2.m[i].any() for i in orc2.ids)
