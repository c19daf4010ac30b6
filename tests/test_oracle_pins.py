"""Pins of the CPU oracle against things other than itself (DESIGN.md §3 pin table).

Closed forms H1/H1b/H2/H3/H4/H5, library routines (torch.optim.AdamW H6, numpy norm H9,
torch bf16 cast), invariants (H7), brute-force shard invariance (H8), exactness of the
reduce (H10), Random123 known-answer vectors (H14).  No value here comes from the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import workloads as W
from oracle import f32

GOLD = os.path.join(os.path.dirname(__file__), "golden")


class G:  # a hyper-parameter group
    def __init__(self, lr=2.0 ** -7, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.0, adapt=1,
                 bias_correction=1):
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.weight_decay, self.adapt, self.bias_correction = weight_decay, adapt, bias_correction


def step1(w, g, grp, t=1, m=None, v=None):
    w = np.array(w, np.float64)
    m = np.zeros_like(w) if m is None else m
    v = np.zeros_like(w) if v is None else v
    st = oracle.lamb_tensor_step(w, m, v, np.array(g, np.float64), grp, t)
    return w, m, v, st


# ---------------------------------------------------------------- H14 Philox KAT
def test_philox_known_answers():
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for ctr, key, exp in kat["vectors"]:
        out = oracle.philox4x32_10([int(x, 16) for x in ctr], [int(x, 16) for x in key])
        assert out == [int(x, 16) for x in exp]


def test_generator_word_keying():
    # element e of tensor i at step s uses word e%4 of Philox(ctr=(e/4 lo, e/4 hi, i, s), key)
    seed = 0x123456789ABCDEF0
    for e in [0, 1, 2, 3, 4, 7, 2**33 + 5]:
        q = e // 4
        key = [seed & 0xFFFFFFFF, (seed >> 32) ^ (2 << 24) ^ 3]
        ctr = [q & 0xFFFFFFFF, q >> 32, 17, 9]
        assert oracle.lib().orc_gen_word(seed, 2, 3, 17, 9, e) == oracle.philox4x32_10(ctr, key)[e % 4]


def test_generator_values_representable():
    w = oracle.gen_weights(W.BASE_SEED, 5, W.INIT_UNIFORM, 200_000)
    assert np.all(w.astype(np.float32).astype(np.float64) == w)      # exact fp32
    assert w.min() >= -1 / 32 and w.max() < 1 / 32
    assert abs(w.std() - (1 / 32) / math.sqrt(3)) < 2e-4            # uniform on [-1/32, 1/32)
    assert np.all(oracle.gen_weights(1, 0, W.INIT_ONE, 10) == 1.0)
    assert np.all(oracle.gen_weights(1, 0, W.INIT_ZERO, 10) == 0.0)
    g = oracle.gen_grads(W.BASE_SEED, 1, 5, 1, W.GEXP_MATRIX, 200_000)
    g32 = torch.from_numpy(g).float()
    assert torch.equal(g32.bfloat16().double(), torch.from_numpy(g))   # exact bf16
    zero = np.mean(g == 0.0)
    assert abs(zero - 1 / 16) < 3e-3
    nz = np.abs(g[g != 0])
    assert nz.min() >= 2.0 ** -13 and nz.max() < 2.0 ** -9
    # different rank terms / steps / tensors give different streams
    assert not np.array_equal(g, oracle.gen_grads(W.BASE_SEED, 2, 5, 1, W.GEXP_MATRIX, 200_000))
    assert not np.array_equal(g, oracle.gen_grads(W.BASE_SEED, 1, 5, 2, W.GEXP_MATRIX, 200_000))


# ---------------------------------------------------------------- closed forms
def test_H1_closed_form():
    w, m, v, (wn, un, ratio) = step1([3.0, 4.0], [1.0, -1.0], G(weight_decay=0.0))
    d = 5.0 / (128.0 * math.sqrt(2.0))
    assert np.allclose(w, [3.0 - d, 4.0 + d], rtol=0, atol=1e-14)
    assert wn == pytest.approx(5.0, abs=1e-14)


def test_H1b_decoupled_decay_inside_norm():
    w, m, v, (wn, un, ratio) = step1([3.0, 4.0], [1.0, -1.0], G(weight_decay=0.5, eps=0.0))
    # u = sign(g) + 0.5 w = [2.5, 1.0]; ||u|| = sqrt(7.25); ratio = 5/sqrt(7.25)
    r = 5.0 / math.sqrt(7.25)
    assert ratio == pytest.approx(r, rel=1e-14)
    assert np.allclose(w, [3.0 - 2.0 ** -7 * r * 2.5, 4.0 - 2.0 ** -7 * r * 1.0], rtol=0, atol=1e-14)


def test_H2_zero_weight_norm_fallback():
    eps = f32(1e-6)
    w, m, v, (wn, un, ratio) = step1([0.0, 0.0, 0.0], [1.0, 2.0, -2.0], G(weight_decay=0.01))
    assert ratio == 1.0 and wn == 0.0
    lr = 2.0 ** -7
    exp = [-lr * 1 / (1 + eps), -lr * 2 / (2 + eps), lr * 2 / (2 + eps)]
    assert np.allclose(w, exp, rtol=1e-14, atol=0)


def test_H3_zero_update_norm_fallback():
    w, m, v, (wn, un, ratio) = step1([1.0, -2.0], [0.0, 0.0], G())
    assert ratio == 1.0 and un == 0.0
    assert list(w) == [1.0, -2.0] and not m.any() and not v.any()


def test_H4_H5_bias_correction_closed_form():
    grp = G()
    w = np.array([1.0]); m = np.zeros(1); v = np.zeros(1)
    b1, b2 = f32(0.9), f32(0.999)
    for t in range(1, 11):
        oracle.lamb_tensor_step(w, m, v, np.array([0.5]), grp, t)
        assert w[0] == pytest.approx((127 / 128) ** t, rel=1e-13)              # H4
        assert m[0] / (1 - b1 ** t) == pytest.approx(0.5, rel=1e-13)            # H5
        assert v[0] / (1 - b2 ** t) == pytest.approx(0.25, rel=1e-12)
    assert w[0] == pytest.approx(0.924565136596599, rel=1e-13)


def test_eps_placement_outside_sqrt():
    # single element, g tiny: r = g/(|g| + eps) (eps outside sqrt) vs g/sqrt(g^2+eps)
    grp = G(adapt=0)
    w, m, v, _ = step1([0.0], [1e-6], grp)
    lr = 2.0 ** -7
    eps = f32(1e-6)
    assert w[0] == pytest.approx(-lr * 1e-6 / (1e-6 + eps), rel=1e-12)


# ---------------------------------------------------------------- H6 AdamW library pin
@pytest.mark.parametrize("wd", [0.0, 0.01, 0.3])
def test_H6_adapt0_equals_torch_adamw(wd):
    rng = np.random.default_rng(7)
    n = 257
    w0 = rng.standard_normal(n) * 0.02
    grp = G(lr=1e-3, weight_decay=wd, adapt=0)
    p = torch.tensor(w0.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.AdamW([p], lr=f32(1e-3), betas=(f32(0.9), f32(0.999)), eps=f32(1e-6),
                            weight_decay=f32(wd))
    w = w0.copy(); m = np.zeros(n); v = np.zeros(n)
    for t in range(1, 11):
        g = rng.standard_normal(n) * 1e-3
        p.grad = torch.tensor(g)
        opt.step()
        oracle.lamb_tensor_step(w, m, v, g, grp, t)
    assert np.max(np.abs(w - p.detach().numpy())) < 1e-13


# ---------------------------------------------------------------- H7 / H9 invariants
def test_H7_step_size_equals_lr_times_weight_norm():
    rng = np.random.default_rng(3)
    grp = G(lr=2.0 ** -10, weight_decay=0.01)
    w = rng.standard_normal(1000) * 0.02; m = np.zeros(1000); v = np.zeros(1000)
    for t in range(1, 6):
        w_before = w.copy()
        wn, un, ratio = oracle.lamb_tensor_step(w, m, v, rng.standard_normal(1000) * 1e-3, grp, t)
        assert np.linalg.norm(w - w_before) == pytest.approx(f32(grp.lr) * np.linalg.norm(w_before),
                                                              rel=1e-12)
        assert wn == pytest.approx(np.linalg.norm(w_before), rel=1e-14)      # H9
        assert ratio == pytest.approx(wn / un, rel=1e-15)


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.standard_normal(100_000) * 0.03,
                        # values exactly halfway between bf16 neighbours (ties to even)
                        (np.arange(1, 2000, dtype=np.float64) * 2 + 1) * 2.0 ** -16 + 1.0])
    ref = torch.from_numpy(x).float().bfloat16().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(oracle.bf16_rne_bits(x), ref)
    for xi in x[:50]:
        assert oracle.lib().orc_bf16_rne(float(xi)) == oracle.bf16_rne_bits(np.array([xi]))[0]


# ---------------------------------------------------------------- H10 exact reduce
@pytest.mark.parametrize("D", [2, 4, 8])
def test_H10_reduced_gradient_exact_in_fp32(D):
    G_ = [oracle.gen_grads(W.BASE_SEED, r + 1, 3, 1, W.GEXP_MATRIX, 50_000) for r in range(D)]
    g = oracle.reduce(G_, 1.0 / D)
    assert np.array_equal(g, np.sum(np.stack(G_), axis=0) / D)
    assert np.array_equal(g.astype(np.float32).astype(np.float64), g)   # representable in fp32


# ---------------------------------------------------------------- H15 bf16 neighbours (Z23, NVLS)
def _bf16_next_up(x):
    t = torch.from_numpy(np.asarray(x, np.float64)).bfloat16()
    return torch.nextafter(t, torch.full_like(t, float("inf"))).double().numpy()


@pytest.mark.parametrize("D", [2, 4, 8])
def test_H15_bf16_neighbors_bracket_the_exact_sum(D):
    # library routines: torch's RNE cast of the exact sum is one of the two neighbours, and the
    # neighbours are adjacent bf16 numbers (torch.nextafter on bf16) bracketing the sum
    G_ = [oracle.gen_grads(W.BASE_SEED, r + 1, 5, 1, W.GEXP_VECTOR, 40_000) for r in range(D)]
    x = oracle.reduce(G_, 1.0)                                   # exact (H10)
    lo, hi = oracle.bf16_neighbors(x)
    rne = torch.from_numpy(x).float().bfloat16().double().numpy()
    assert np.all((rne == lo) | (rne == hi))
    assert np.all(lo <= x) and np.all(x <= hi)
    exact = lo == hi
    assert np.array_equal(lo[exact], x[exact])
    assert np.array_equal(_bf16_next_up(lo[~exact]), hi[~exact])
    assert 0 < exact.sum() < x.size                              # both kinds occur


def test_H15_bf16_neighbors_special_cases():
    x = np.array([1.0, 1.0 + 2.0 ** -8, -(1.0 + 2.0 ** -8), -1.5, 2.0 ** -126 * (1 + 2.0 ** -10), 0.0])
    lo, hi = oracle.bf16_neighbors(x)
    assert list(lo) == [1.0, 1.0, -(1.0 + 2.0 ** -7), -1.5, 2.0 ** -126, 0.0]
    assert list(hi) == [1.0, 1.0 + 2.0 ** -7, -1.0, -1.5, 2.0 ** -126 * (1 + 2.0 ** -7), 0.0]


# ---------------------------------------------------------------- H8 shard invariance
def _flat_state(wl, pl):
    n = pl.flat_size
    w = np.zeros(n); g = np.zeros(n)
    for i, ts in enumerate(wl.tensors):
        o = pl.tensor_off[i]
        w[o:o + ts.numel] = oracle.gen_weights(wl.seed, i, ts.init, ts.numel)
    return w, g


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_H8_shard_count_invariance(seed):
    rng = np.random.default_rng(seed)
    tensors = W.random_table(rng, 12, max_numel=700, p_big=0.2, big=3000)
    wl = W.Workload("rand", 9, tensors, W.default_groups(lr=2.0 ** -7))
    ref = oracle.OracleRun(wl, world_size=1, mode=oracle.REPLICATED)
    for t in (1, 2):
        ref.step(t)
    for S in range(1, 9):
        pl = oracle.plan([t.numel for t in tensors], S, cap=2048)
        w, g = _flat_state(wl, pl)
        m = np.zeros_like(w); v = np.zeros_like(w)
        for t in (1, 2):
            g[:] = 0
            for i, ts in enumerate(tensors):
                o = pl.tensor_off[i]
                g[o:o + ts.numel] = ref.grads(i, t)
            stats = oracle.sharded_step(wl, pl, w, m, v, g, t)
        for i, ts in enumerate(tensors):
            o = pl.tensor_off[i]
            assert np.allclose(w[o:o + ts.numel], ref.w[i], rtol=1e-13, atol=1e-16)
            assert np.allclose(m[o:o + ts.numel], ref.m[i], rtol=1e-13, atol=1e-18)
            assert stats[i][2] == pytest.approx(ref.stats[i][2], rel=1e-13)
        if S > 1:
            assert pl.straddlers, "case should exercise straddlers"
