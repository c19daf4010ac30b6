"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
inputs.  Needs a B200; run with `pytest -m gpu`."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W
from gpu_common import compare_state, run_gpu, snapshot_w, spec_of

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]
GOLD = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lamb():
    from paper_2402_15627_b200 import build
    build.build()
    from paper_2402_15627_b200 import lamb as L
    print(f"[lib] {L.LIB_PATH}", flush=True)
    return L


def test_device_philox_known_answers(lamb):
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for ctr, key, exp in kat["vectors"]:
        assert lamb.device_philox([int(x, 16) for x in ctr], [int(x, 16) for x in key]) == \
            [int(x, 16) for x in exp]


def test_generator_matches_oracle_bit_exact(lamb):
    wl = W.toy()
    L = run_gpu(wl, steps=0)
    L.synth_grads(spec_of(wl), wl.seed, 1, 3)
    g = L.grad_buffer().float().cpu().numpy().astype(np.float64)
    w = L.get_state(lamb.LAMB_BUF_W).astype(np.float64)
    for i, ts in enumerate(wl.tensors):
        o = int(L.plan.tensor_off[i])
        assert np.array_equal(g[o:o + ts.numel], oracle.gen_grads(wl.seed, 1, i, 3, ts.gexp, ts.numel))
        assert np.array_equal(w[o:o + ts.numel], oracle.gen_weights(wl.seed, i, ts.init, ts.numel))
        end = int(L.plan.tensor_off[i + 1]) if i + 1 < len(wl.tensors) else L.plan.flat_size
        assert not g[o + ts.numel:end].any()          # padding stays zero
    L.close()


@pytest.mark.parametrize("lr", [2.0 ** -10, 2.0 ** -7])
@pytest.mark.parametrize("steps", [1, 10])
def test_toy_parity(lamb, steps, lr):
    """BASELINE configs[0] at the bench lr and at the hand-case lr: w, m, v, params, ratios and
    the last step's per-element update against the oracle."""
    wl = W.toy()
    wl.groups = W.default_groups(lr=lr)
    L = run_gpu(wl, steps=steps)
    orc = oracle.OracleRun(wl, world_size=1, mode=oracle.PER_RANK)
    for t in range(1, steps + 1):
        orc.step(t)
    compare_state(L, orc, steps)
    print(f"toy steps={steps} lr={lr}: update check max |err|/allowed = {L.update_worst:.3f}")
    assert 0.0 < L.update_worst <= 1.0
    L.close()


@pytest.mark.parametrize("seed", range(4))
def test_random_ragged_tables(lamb, seed):
    rng = np.random.default_rng(500 + seed)
    tensors = W.random_table(rng, 40, max_numel=3000, p_big=0.15, big=60_000)
    tensors.append(W.TensorSpec("one", 1, W.NO_DECAY, W.INIT_UNIFORM, W.GEXP_VECTOR))
    wl = W.Workload("rand", 20 + seed, tensors, W.default_groups(lr=2.0 ** -7))
    cap = int(rng.choice([1, 4096, 20_000]))
    L = run_gpu(wl, steps=3, cap=cap)
    orc = oracle.OracleRun(wl, world_size=1)
    for t in (1, 2, 3):
        orc.step(t)
    compare_state(L, orc, 3)
    L.close()


def test_group_variants(lamb):
    """adapt=0 (AdamW), no bias correction, lr=0, large weight decay."""
    rng = np.random.default_rng(9)
    tensors = [W.TensorSpec(f"x{k}", int(rng.integers(1, 9000)), k, W.INIT_UNIFORM, W.GEXP_MATRIX)
               for k in range(4)]
    groups = [W.GroupSpec(lr=2.0 ** -7, weight_decay=0.01, adapt=0),
              W.GroupSpec(lr=2.0 ** -7, weight_decay=0.0, bias_correction=0),
              W.GroupSpec(lr=0.0, weight_decay=0.01),
              W.GroupSpec(lr=2.0 ** -8, weight_decay=0.5, beta1=0.8, beta2=0.99, eps=1e-8)]
    wl = W.Workload("groups", 30, tensors, groups)
    L = run_gpu(wl, steps=4)
    orc = oracle.OracleRun(wl, world_size=1)
    for t in range(1, 5):
        orc.step(t)
    compare_state(L, orc, 4)
    L.close()


@pytest.mark.parametrize("seed", range(6))
def test_random_hyperparameters_property(lamb, seed):
    """Property sweep (SPEC-style randomized small configs): random ragged tables under random
    groups — beta1 in [0.5, 0.99), beta2 in [0.9, 0.9999), eps in [1e-9, 1e-4], weight decay in
    [0, 0.3], lr a power of two in [2^-12, 2^-6], adapt / bias correction on or off, a random
    bucket cap — 1-3 steps, element-wise against the oracle with the per-step update check."""
    rng = np.random.default_rng(1000 + seed)
    n_groups = int(rng.integers(1, 5))
    groups = [W.GroupSpec(lr=2.0 ** -int(rng.integers(6, 13)), beta1=float(np.float32(rng.uniform(0.5, 0.99))),
                          beta2=float(np.float32(rng.uniform(0.9, 0.9999))),
                          eps=float(np.float32(10.0 ** rng.uniform(-9, -4))),
                          weight_decay=float(np.float32(rng.uniform(0, 0.3))) if rng.random() < 0.7 else 0.0,
                          adapt=int(rng.random() < 0.8), bias_correction=int(rng.random() < 0.8))
              for _ in range(n_groups)]
    tensors = W.random_table(rng, int(rng.integers(5, 40)), max_numel=6000, p_big=0.2, big=60_000)
    tensors = [W.TensorSpec(t.name, t.numel, int(rng.integers(0, n_groups)), t.init, t.gexp) for t in tensors]
    wl = W.Workload("prop", 40 + seed, tensors, groups)
    steps = int(rng.integers(1, 4))
    L = run_gpu(wl, steps=steps, cap=int(rng.integers(2000, 80_000)))
    orc = oracle.OracleRun(wl, world_size=1)
    for t in range(1, steps + 1):
        orc.step(t)
    compare_state(L, orc, steps)
    print(f"seed {seed}: {len(tensors)} tensors, {n_groups} groups, {steps} steps, "
          f"update check max |err|/allowed = {L.update_worst:.3f}")
    L.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_devices_in_one_process(lamb):
    """Handles on two GPUs in one process (lamb.h: several handles per process): the
    shared-memory opt-in of the TMA passes is per device, so the second device's launches run
    too, and both devices give bitwise-identical results on the same inputs."""
    rng = np.random.default_rng(78)
    wl = W.Workload("two", 41, W.random_table(rng, 20, max_numel=30000), W.default_groups())
    outs = []
    for dev in (0, 1):
        L = run_gpu(wl, steps=2, cap=50_000, device=dev)
        outs.append([L.get_state(k) for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V)]
                    + [L.param_buffer().view(torch.int16).cpu().numpy()])
        L.close()
    for a, b in zip(*outs):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    orc = oracle.OracleRun(wl)
    for t in (1, 2):
        orc.step(t)
    L = run_gpu(wl, steps=2, cap=50_000, device=1)
    compare_state(L, orc, 2)
    L.close()


def test_determinism_bitwise(lamb):
    """H13: two runs give bitwise-identical w, m, v, params (no float atomics)."""
    rng = np.random.default_rng(77)
    wl = W.Workload("det", 40, W.random_table(rng, 30, max_numel=20000), W.default_groups())
    outs = []
    for _ in range(2):
        L = run_gpu(wl, steps=3, cap=50_000)
        outs.append([L.get_state(k) for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V)]
                    + [L.param_buffer().view(torch.int16).cpu().numpy()])
        L.close()
    for a, b in zip(*outs):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_zero_grad_tensor_and_zero_weights(lamb):
    """Z9 fallbacks on the GPU: ||w|| = 0 (zero-init biases at step 1) and ||u|| = 0."""
    tensors = [W.TensorSpec("zb", 100, W.NO_DECAY, W.INIT_ZERO, W.GEXP_VECTOR),
               W.TensorSpec("m", 4096, W.DECAY, W.INIT_UNIFORM, W.GEXP_MATRIX)]
    wl = W.Workload("z", 41, tensors, W.default_groups(lr=2.0 ** -7))
    L = run_gpu(wl, steps=1)
    _, _, ratio = L.tensor_stats()
    assert ratio[0] == 1.0
    orc = oracle.OracleRun(wl)
    orc.step(1)
    compare_state(L, orc, 1)
    # ||u|| = 0: zero grads and zero decay -> unchanged weights, ratio 1
    L.grad_buffer().zero_()
    wl2 = W.Workload("z2", 42, [W.TensorSpec("a", 1000, 0, W.INIT_UNIFORM, W.GEXP_VECTOR)],
                     [W.GroupSpec(weight_decay=0.0)])
    L2 = run_gpu(wl2, steps=0)
    w0 = L2.get_state(lamb.LAMB_BUF_W).copy()
    L2.step(1)
    torch.cuda.synchronize()
    assert np.array_equal(L2.get_state(lamb.LAMB_BUF_W), w0)
    assert L2.tensor_stats()[2][0] == 1.0
    L.close()
    L2.close()


def test_abi_errors_on_gpu(lamb):
    wl = W.toy()
    L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups)
    with pytest.raises(lamb.LambError) as e:
        L.step(1)                      # master not set
    assert e.value.status == lamb.LAMB_ESTATE
    L.synth_init(spec_of(wl), wl.seed)
    with pytest.raises(lamb.LambError) as e:
        L.step(0)
    assert e.value.status == lamb.LAMB_EINVAL
    L.close()


def test_set_master_and_step_host(lamb):
    """lamb_set_master from a host array + the host-buffer e2e entry point."""
    wl = W.toy()
    L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups)
    flat = torch.zeros(L.plan.flat_size, dtype=torch.float32)
    orc = oracle.OracleRun(wl)
    for i, ts in enumerate(wl.tensors):
        o = int(L.plan.tensor_off[i])
        flat[o:o + ts.numel] = torch.from_numpy(orc.w[i]).float()
    L.set_master(flat)
    L.w_prev = snapshot_w(L)
    L.synth_grads(spec_of(wl), wl.seed, 1, 1)
    hg = L.grad_buffer().cpu().pin_memory()
    hp = torch.empty(L.plan.flat_size, dtype=torch.bfloat16).pin_memory()
    L.grad_buffer().zero_()
    L.step_host(hg, hp, 1)
    torch.cuda.synchronize()
    orc.step(1)
    compare_state(L, orc, 1)
    assert torch.equal(hp.view(torch.int16), L.param_buffer().cpu().view(torch.int16))
    L.close()


def test_gpt13b_layout_1p3b_full_size_sampled(lamb):
    """BASELINE configs[1] at full size in the bench launch configuration: sampled tensors
    against the oracle (every tensor's result depends only on its own data), and the
    step-size invariant ||dw|| = lr ||w|| (H7) on every adapted tensor."""
    wl = W.gpt_1p3b()
    from paper_2402_15627_b200 import lamb as Lm
    L = Lm.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, timing=True)
    spec = spec_of(wl)
    L.synth_init(spec, wl.seed)
    L.synth_grads(spec, wl.seed, 1, 1)
    w_before = L.state_buffer(Lm.LAMB_BUF_W).clone()
    ids = [0] + list(range(1, 13)) + [len(wl.tensors) - 2, len(wl.tensors) - 1]
    L.w_prev = snapshot_w(L, ids)
    L.step(1)
    torch.cuda.synchronize()
    w_after = L.state_buffer(Lm.LAMB_BUF_W)
    orc = oracle.OracleRun(wl, world_size=1, tensor_ids=ids)
    orc.step(1)
    compare_state(L, orc, 1, ids=ids)
    # H7 on every tensor, computed with torch on the device from the library's state
    lr = float(np.float32(W.LR_BENCH))
    for (i, soff, toff, ln) in L.plan.segments.tolist():
        a = w_before[soff:soff + ln].double()
        b = w_after[soff:soff + ln].double()
        wn = torch.linalg.vector_norm(a).item()
        if wn == 0.0:
            continue
        dn = torch.linalg.vector_norm(b - a).item()
        assert abs(dn - lr * wn) <= 2e-5 * lr * wn + 1e-9, (i, dn, lr * wn)
    L.close()


@pytest.mark.parametrize("case", ["toy", "ragged-buckets", "mixed-whole"])
def test_step_host_pipeline_matches_device_steps(lamb, case):
    """lamb_step_host over several consecutive steps (per-bucket pipeline: uploads of step t+1
    overlapping the LAMB work and the downloads of step t) is bit-identical to lamb_step on
    device-resident grads.  "mixed-whole": steps with the pre-step enabled take the whole-step
    pipeline, interleaved with per-bucket steps."""
    if case == "toy":
        wl, cap = W.toy(), 0
    else:
        rng = np.random.default_rng(29)
        wl = W.Workload("hb", 73, W.random_table(rng, 40, max_numel=7000, p_big=0.2, big=40_000),
                        W.default_groups(lr=2.0 ** -7))
        cap = 10_000
    spec = spec_of(wl)
    n = 5
    A = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, bucket_cap=cap)
    B = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, bucket_cap=cap)
    if case != "toy":
        assert A.plan.buckets.shape[0] > 4
    A.synth_init(spec, wl.seed)
    B.synth_init(spec, wl.seed)
    hg = [torch.empty(A.plan.flat_size, dtype=torch.bfloat16).pin_memory() for _ in range(n)]
    hp = [torch.empty(A.plan.flat_size, dtype=torch.bfloat16).pin_memory() for _ in range(n)]
    for t in range(1, n + 1):
        A.synth_grads(spec, wl.seed, 1, t)
        hg[t - 1].copy_(A.grad_buffer())
    torch.cuda.synchronize()
    A.grad_buffer().zero_()
    clip_at = {3} if case == "mixed-whole" else set()
    for t in range(1, n + 1):
        A.set_grad_clip(0.05 if t in clip_at else 0.0)
        A.step_host(hg[t - 1], hp[t - 1], t)        # no sync between calls
    torch.cuda.synchronize()
    for t in range(1, n + 1):
        B.synth_grads(spec, wl.seed, 1, t)
        B.set_grad_clip(0.05 if t in clip_at else 0.0)
        B.step(t)
        torch.cuda.synchronize()
        assert torch.equal(hp[t - 1].view(torch.int16), B.param_buffer().cpu().view(torch.int16)), t
    for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V):
        assert np.array_equal(A.get_state(k).view(np.uint32), B.get_state(k).view(np.uint32))
    A.close()
    B.close()


def test_checkpoint_resume_and_reshard(lamb, tmp_path):
    """NEXT #4: two-stage save at step 3; resume in the same layout is bit-identical to an
    uninterrupted run; resume into a different bucket layout (reshard) matches the oracle;
    the file holds the oracle's state (independent numpy reader)."""
    from ckpt_reader import read_checkpoint
    rng = np.random.default_rng(17)
    tensors = W.random_table(rng, 25, max_numel=6000, p_big=0.2, big=40_000)
    wl = W.Workload("ck", 70, tensors, W.default_groups(lr=2.0 ** -7))
    spec = spec_of(wl)
    path = str(tmp_path / "lamb.ckpt")
    A = run_gpu(wl, steps=3, cap=10_000)
    A.checkpoint_save(path, 3)
    for t in (4, 5):                      # training continues while stage 2 writes
        A.synth_grads(spec, wl.seed, 1, t)
        A.step(t)
    A.checkpoint_wait()
    torch.cuda.synchronize()
    orc = oracle.OracleRun(wl)
    for t in (1, 2, 3):
        orc.step(t)
    ck = read_checkpoint(path)
    assert ck["step"] == 3 and list(ck["numel"]) == [t.numel for t in tensors]
    for i in range(len(tensors)):
        for name, ref in (("w", orc.w[i]), ("m", orc.m[i]), ("v", orc.v[i])):
            x = ck[name][i].astype(np.float64)
            atol = 1e-6 if name == "w" else 1e-6 * np.max(np.abs(ref))
            assert np.all(np.abs(x - ref) <= atol + 1e-4 * np.abs(ref)), (i, name)
    for cap in (10_000, 3_000):           # same layout, then a different one
        B = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=cap)
        assert B.checkpoint_load(path) == 3
        for t in (4, 5):
            B.synth_grads(spec, wl.seed, 1, t)
            B.step(t)
        torch.cuda.synchronize()
        if cap == 10_000:
            for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V):
                assert np.array_equal(A.get_state(k).view(np.uint32), B.get_state(k).view(np.uint32))
            assert torch.equal(A.param_buffer().view(torch.int16), B.param_buffer().view(torch.int16))
        else:
            orc2 = oracle.OracleRun(wl)
            for t in range(1, 6):
                orc2.step(t)
            compare_state(B, orc2, 5)
        B.close()
    with pytest.raises(lamb.LambError):   # a different parameter table is refused
        C = lamb.Lamb([(10, 0)], wl.groups)
        C.checkpoint_load(path)
    # a failed background write is reported once by the next wait, then a save works again
    A.checkpoint_save(str(tmp_path / "no_such_dir" / "x.ckpt"), 5)
    with pytest.raises(lamb.LambError, match="open"):
        A.checkpoint_wait()
    A.checkpoint_wait()
    A.checkpoint_save(str(tmp_path / "again.ckpt"), 5)
    A.checkpoint_wait()
    assert read_checkpoint(str(tmp_path / "again.ckpt"))["step"] == 5
    A.close()


@pytest.mark.parametrize("frac,inv_scale", [(0.25, 1.0), (10.0, 1.0), (0.5, 2.0 ** -10)])
def test_prestep_clip_and_loss_scale(lamb, frac, inv_scale):
    """NEXT #3 on the GPU: global grad-norm clipping (clip active / inactive) and loss-scale
    unscaling against the oracle's pre-step; reported norm and clip coefficient match."""
    rng = np.random.default_rng(31)
    tensors = W.random_table(rng, 30, max_numel=6000, p_big=0.2, big=40_000)
    wl = W.Workload("clip", 90, tensors, W.default_groups(lr=2.0 ** -7))
    spec = spec_of(wl)
    S = 1.0 / inv_scale
    orc = oracle.OracleRun(wl)
    gn1 = np.sqrt(sum(np.sum(orc.grads(i, 1) ** 2) for i in orc.ids))
    max_norm = float(np.float32(frac * gn1))
    if S != 1.0:   # feed loss-scaled grads S * g (exact in bf16 for a power of two)
        orig = orc.grads
        orc.grads = lambda i, t: orig(i, t) * S
    L = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=20_000)
    L.synth_init(spec, wl.seed)
    L.set_grad_clip(max_norm)
    L.set_loss_scale(inv_scale)
    for t in (1, 2, 3):
        L.synth_grads(spec, wl.seed, 1, t)
        L.w_prev = snapshot_w(L)
        if S != 1.0:
            g = L.grad_buffer()
            g.copy_((g.float() * S).bfloat16())
        L.step(t)
        info = orc.step(t, max_grad_norm=max_norm, inv_loss_scale=inv_scale)
        gi = L.step_info()
        assert not gi["skipped"]
        assert gi["grad_norm"] == pytest.approx(info["grad_norm"], rel=1e-6)
        assert gi["clip"] == pytest.approx(info["clip"], rel=1e-6)
        if frac < 1:
            assert info["clip"] < 1.0
    compare_state(L, orc, 3)
    L.close()


def test_prestep_nonfinite_skip(lamb):
    wl = W.toy()
    spec = spec_of(wl)
    L = run_gpu(wl, steps=1)
    L.set_grad_clip(1.0)
    before = [L.get_state(k).copy() for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V)]
    p0 = L.param_buffer().clone()
    L.synth_grads(spec, wl.seed, 1, 2)
    L.grad_buffer()[100] = float("inf")
    L.step(2)
    info = L.step_info()
    assert info["skipped"]
    after = [L.get_state(k) for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V)]
    for a, b in zip(before, after):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert torch.equal(p0.view(torch.int16), L.param_buffer().view(torch.int16))
    L.synth_grads(spec, wl.seed, 1, 2)     # next step with finite grads proceeds
    L.step(2)
    assert not L.step_info()["skipped"]
    L.close()


@pytest.mark.parametrize("defer", [False, True])
def test_step_bucket_equals_step(lamb, defer):
    """NEXT #2: stepping every bucket in backward (reverse) order is bit-identical to one
    lamb_step (per-bucket LAMB is exact: a tensor never spans buckets)."""
    rng = np.random.default_rng(55)
    tensors = W.random_table(rng, 40, max_numel=6000, p_big=0.2, big=40_000)
    wl = W.Workload("bk", 95, tensors, W.default_groups(lr=2.0 ** -7))
    spec = spec_of(wl)
    A = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=15_000)
    B = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=15_000)
    nb = len(A.plan.buckets)
    assert nb > 3
    for L in (A, B):
        L.synth_init(spec, wl.seed)
    for t in (1, 2, 3):
        for L in (A, B):
            L.synth_grads(spec, wl.seed, 1, t)
        A.step(t)
        if t == 3:
            B.w_prev = snapshot_w(B)
        for b in reversed(range(nb)):
            B.step_bucket(b, t, defer_ag=defer)
        if defer:
            for b in range(nb):
                B.gather_bucket(b)
    torch.cuda.synchronize()
    for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V):
        assert np.array_equal(A.get_state(k).view(np.uint32), B.get_state(k).view(np.uint32))
    assert torch.equal(A.param_buffer().view(torch.int16), B.param_buffer().view(torch.int16))
    orc = oracle.OracleRun(wl)          # the per-bucket path against the oracle itself
    for t in (1, 2, 3):
        orc.step(t)
    compare_state(B, orc, 3)
    B.set_grad_clip(1.0)
    with pytest.raises(lamb.LambError) as e:
        B.step_bucket(0, 4)
    assert e.value.status == lamb.LAMB_EUNSUPPORTED
    A.close()
    B.close()


def test_results_independent_of_grid_and_sm_partition(lamb):
    """Determinism does not depend on the launch configuration: per-item partials are fixed
    reductions whatever warp runs the item, so any SM budget (lamb_set_max_ctas) or a green-
    context SM partition gives bit-identical state."""
    rng = np.random.default_rng(61)
    tensors = W.random_table(rng, 40, max_numel=20000, p_big=0.2, big=200_000)
    wl = W.Workload("grid", 96, tensors, W.default_groups(lr=2.0 ** -7))
    spec = spec_of(wl)
    outs = []
    for mode in ("full", "ctas7", "ctas148", "green"):
        L = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=100_000)
        L.synth_init(spec, wl.seed)
        stream = None
        if mode.startswith("ctas"):
            L.set_max_ctas(int(mode[4:]))
        if mode == "green":
            lp, _, got = lamb.sm_partition(0, 16)
            assert 16 <= got < 148
            stream = torch.cuda.ExternalStream(lp)
            L.set_max_ctas(2 * got)
        for t in (1, 2):
            L.synth_grads(spec, wl.seed, 1, t)
            L.step(t, stream=stream)
        torch.cuda.synchronize()
        outs.append([L.get_state(k).view(np.uint32) for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V)]
                    + [L.param_buffer().view(torch.int16).cpu().numpy()])
        L.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def test_cuda_graph_step_equals_eager(lamb):
    """a7: LAMB_FLAG_GRAPH replays one captured graph of the step (constants refreshed by the
    prologue each step); bit-identical to eager launches, also after a re-capture when the
    pre-step is switched on."""
    rng = np.random.default_rng(67)
    tensors = W.random_table(rng, 30, max_numel=20000, p_big=0.2, big=100_000)
    wl = W.Workload("graph", 97, tensors, W.default_groups(lr=2.0 ** -7))
    spec = spec_of(wl)
    E = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=50_000)
    G = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=50_000, graph=True)
    for L in (E, G):
        L.synth_init(spec, wl.seed)
    for t in range(1, 6):
        if t == 4:
            for L in (E, G):
                L.set_grad_clip(0.05)
        for L in (E, G):
            L.synth_grads(spec, wl.seed, 1, t)
            L.step(t)
    torch.cuda.synchronize()
    for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V):
        assert np.array_equal(E.get_state(k).view(np.uint32), G.get_state(k).view(np.uint32))
    assert torch.equal(E.param_buffer().view(torch.int16), G.param_buffer().view(torch.int16))
    assert G.step_info()["clip"] < 1.0
    E.close()
    G.close()


def test_cuda_graph_follows_changed_clip_and_loss_scale(lamb):
    """the pre-step scalars (max_grad_norm, inv_loss_scale) are passed to the graph's
    kernels by value, so changing them from one non-default value to another must re-capture;
    eager and graph handles stay bitwise equal while both change every step."""
    rng = np.random.default_rng(71)
    tensors = W.random_table(rng, 20, max_numel=20000, p_big=0.2, big=60_000)
    wl = W.Workload("graphclip", 99, tensors, W.default_groups(lr=2.0 ** -7))
    spec = spec_of(wl)
    E = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=50_000)
    G = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=50_000, graph=True)
    for L in (E, G):
        L.synth_init(spec, wl.seed)
    settings = [(0.05, 1.0), (0.02, 1.0), (0.02, 0.5), (0.08, 0.25), (0.0, 0.25)]
    for t, (clip, inv) in enumerate(settings, start=1):
        for L in (E, G):
            L.set_grad_clip(clip)
            L.set_loss_scale(inv)
            L.synth_grads(spec, wl.seed, 1, t)
            L.step(t)
        torch.cuda.synchronize()
        ie, ig = E.step_info(), G.step_info()
        assert ie["clip"] == ig["clip"] and ie["grad_norm"] == ig["grad_norm"], (t, ie, ig)
        for k in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V):
            assert np.array_equal(E.get_state(k).view(np.uint32), G.get_state(k).view(np.uint32)), t
    E.close()
    G.close()


def test_max_size_tensor_beyond_int32(lamb):
    """Maximum-size edge case: one tensor of 2^31 + 3 elements (flat, shard and in-tensor
    offsets beyond int32; 537k work items in one segment) next to a 1-element tensor, one
    step, every element against the oracle."""
    big = 2 ** 31 + 3
    tensors = [W.TensorSpec("huge", big, W.DECAY, W.INIT_UNIFORM, W.GEXP_MATRIX),
               W.TensorSpec("one", 1, W.NO_DECAY, W.INIT_ONE, W.GEXP_VECTOR)]
    wl = W.Workload("max", 98, tensors, W.default_groups(lr=2.0 ** -7))
    L = run_gpu(wl, steps=1, cap=0)
    assert L.plan.flat_size > 2 ** 31
    orc = oracle.OracleRun(wl)
    orc.step(1)
    compare_state(L, orc, 1, ids=[0, 1], check_params=False)
    p = L.param_buffer()
    for lo in (0, 2 ** 31 - 8, big - 8):          # params around the int32 boundary and the end
        got = p[lo:lo + 8].view(torch.int16).cpu().numpy().view(np.uint16)
        w = L.state_buffer(lamb.LAMB_BUF_W)[lo:lo + 8].cpu().numpy().astype(np.float64)
        assert np.array_equal(got, oracle.bf16_rne_bits(w))
    L.close()


def test_torch_optimizer_binding_end_to_end(lamb):
    """LambOptimizer drives lamb_step from a real PyTorch loop (bf16 MLP): params are views of
    the library's param buffer, autograd accumulates into its grad buffer; three iterations
    against the oracle fed the same captured gradients (exact bf16 values, D = 1)."""
    from paper_2402_15627_b200.torch_optim import LambOptimizer
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(96, 200), torch.nn.GELU(), torch.nn.Linear(200, 33)).cuda().bfloat16()
    weights = [p for n, p in model.named_parameters() if p.dim() > 1]
    biases = [p for n, p in model.named_parameters() if p.dim() == 1]
    groups = [{"params": weights, "weight_decay": 0.01}, {"params": biases, "weight_decay": 0.0}]
    ordered = weights + biases
    w0 = [p.detach().double().cpu().numpy().reshape(-1).copy() for p in ordered]
    opt = LambOptimizer(groups, lr=2.0 ** -7, betas=(0.9, 0.999), eps=1e-6)
    x = torch.randn(64, 96, device="cuda", dtype=torch.bfloat16)
    grads = []
    for _ in range(3):
        opt.zero_grad()
        model(x).float().pow(2).mean().backward()
        grads.append([p.grad.detach().double().cpu().numpy().reshape(-1).copy() for p in ordered])
        opt.step()
    torch.cuda.synchronize()
    # the oracle, tensor by tensor, on the captured gradients
    class Grp:
        def __init__(self, wd):
            self.lr, self.beta1, self.beta2, self.eps = 2.0 ** -7, 0.9, 0.999, 1e-6
            self.weight_decay, self.adapt, self.bias_correction = wd, 1, 1
    state = []
    for k, wk in enumerate(w0):
        grp = Grp(0.01 if k < len(weights) else 0.0)
        w, m, v = wk.copy(), np.zeros_like(wk), np.zeros_like(wk)
        for t in range(3):
            oracle.lamb_tensor_step(w, m, v, grads[t][k], grp, t + 1)
        state.append((w, m, v))
    Wg, Mg, Vg = (opt.L.get_state(b) for b in (lamb.LAMB_BUF_W, lamb.LAMB_BUF_M, lamb.LAMB_BUF_V))
    for (i, soff, toff, ln) in opt.L.plan.segments.tolist():
        w, m, v = state[i]
        for got, ref in ((Wg, w), (Mg, m), (Vg, v)):
            g = got[soff:soff + ln].astype(np.float64)
            r = ref[toff:toff + ln]
            atol = 1e-6 if ref is w else 1e-6 * np.max(np.abs(ref))
            assert np.all(np.abs(g - r) <= atol + 1e-4 * np.abs(r)), i
        # the model's parameter IS bf16_rne of the master
        pb = ordered[i].detach().reshape(-1)[toff:toff + ln].view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(pb, oracle.bf16_rne_bits(Wg[soff:soff + ln].astype(np.float64)))
    opt.L.close()


def test_self_check_detects_corruption(lamb):
    """lamb_self_check (§4.3-style diagnostic): healthy state reads all-zero; a NaN in
    m, a stale param, nonzero shard padding and a write outside a tensor view are each found."""
    wl = W.toy()
    L = run_gpu(wl, steps=2)
    assert all(v == 0 for v in L.self_check().values())
    tail = int(L.plan.tensor_off[0]) + wl.tensors[0].numel          # padding after tensor 0? (3072 is 8-aligned)
    flat_pad = int(L.plan.tensor_off[1]) + wl.tensors[1].numel      # t1 = 48 elements -> next start 3120: no gap
    flat_pad = int(L.plan.tensor_off[2]) + wl.tensors[2].numel      # end of t2 .. flat_size is padding
    L.grad_buffer()[flat_pad + 3] = 1.0
    L.state_buffer(lamb.LAMB_BUF_M)[17] = float("nan")
    L.param_buffer()[5] = 123.0
    L.state_buffer(lamb.LAMB_BUF_V)[L.plan.shard_size - 1] = 1.0   # last shard element is padding
    torch.cuda.synchronize()
    c = L.self_check()
    assert c["nonfinite_state"] >= 1 and c["param_mismatch"] >= 1
    assert c["shard_padding_nonzero"] >= 1 and c["flat_padding_nonzero"] >= 1
    assert c["peer_unreachable"] == 0
    L.close()


def test_copy_engine_schedule_needs_the_flag(lamb):
    """lamb_push_grads_bucket / lamb_step_staged / lamb_wait_params_bucket on a handle without
    LAMB_FLAG_CE (here D = 1) fail with EUNSUPPORTED and leave the handle usable."""
    wl = W.toy()
    L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups)
    L.synth_init(spec_of(wl), wl.seed)
    for call in (lambda: L.push_grads_bucket(0, 1), lambda: L.step_staged(1), lambda: L.wait_params_bucket(0, 1)):
        with pytest.raises(lamb.LambError) as ei:
            call()
        assert ei.value.status == lamb.LAMB_EUNSUPPORTED
    L.synth_grads(spec_of(wl), wl.seed, 1, 1)
    L.step(1)
    torch.cuda.synchronize()
    L.close()


def test_checkpoint_commit_protocol(lamb, tmp_path):
    """saves go to path.tmp.<n> and are renamed only once every rank committed its
    partition; a failed save leaves the previous checkpoint at `path` intact; a file with a
    missing commit word (a partition that never completed) is refused by load."""
    from ckpt_reader import read_checkpoint
    wl = W.toy()
    spec = spec_of(wl)
    path = str(tmp_path / "c.ckpt")
    L = run_gpu(wl, steps=2)
    L.checkpoint_save(path, 2)
    L.checkpoint_wait()
    assert os.path.exists(path) and not [f for f in os.listdir(tmp_path) if ".tmp." in f]
    ck = read_checkpoint(path)
    assert ck["step"] == 2 and ck["world"] == 1 and ck["commit"][0] != 0
    good = open(path, "rb").read()
    # a save that fails (its temporary cannot be created: a directory is in the way, which
    # stops root too) must not touch the previous file
    L.synth_grads(spec, wl.seed, 1, 3)
    L.step(3)
    os.mkdir(path + ".tmp.1")                # the handle's second save writes path.tmp.1
    L.checkpoint_save(path, 3)
    with pytest.raises(lamb.LambError, match="open"):
        L.checkpoint_wait()
    assert open(path, "rb").read() == good
    # a missing commit word: refused
    bad = bytearray(good)
    off = 64 + 8 * len(wl.tensors)
    bad[off:off + 8] = bytes(8)
    bpath = str(tmp_path / "bad.ckpt")
    open(bpath, "wb").write(bytes(bad))
    B = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups)
    with pytest.raises(lamb.LambError, match="incomplete"):
        B.checkpoint_load(bpath)
    assert B.checkpoint_load(path) == 2
    B.close()
    L.close()


def test_set_master_from_host_needs_one_bucket_of_device_memory(lamb):
    """lamb_set_master from host memory stages bucket by bucket through one
    bucket-sized device buffer.  175B-slice-3L layout (BASELINE configs[3]'s layer shape,
    5.4B params, 87 GB of state at D = 1): after create, a ballast leaves less free device
    memory than a flat_size fp32 temporary (21.7 GB) but more than one bucket (160 MB); the
    host round trip W = set_master(x) must succeed and read back exactly."""
    wl = W.slice_175b(3)
    L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, bucket_cap=wl.cap)
    n = L.plan.flat_size
    max_bucket = int(L.plan.buckets[:, 1].max())
    free, _ = torch.cuda.mem_get_info()
    keep = 4 * max_bucket + (2 << 30)        # one bucket + 2 GiB of headroom for the runtime
    ballast = torch.empty(max(0, free - keep), dtype=torch.uint8, device="cuda")
    assert torch.cuda.mem_get_info()[0] < 4 * n           # a flat fp32 temporary cannot fit
    x = torch.empty(n, dtype=torch.float32, pin_memory=True)
    gen = torch.Generator().manual_seed(5)
    x.copy_(torch.randn(n, generator=gen))
    mask = torch.zeros(n, dtype=torch.bool)
    for t, off in zip(wl.tensors, L.plan.tensor_off.tolist()):
        mask[off:off + t.numel] = True
    x[~mask] = 0
    L.set_master(x)
    w = L.state_buffer(lamb.LAMB_BUF_W)
    assert torch.equal(w.cpu(), x), "w != the host master (D = 1: the shard is the flat array)"
    p = L.param_buffer()
    for lo in (0, n // 2, n - 4096):
        assert torch.equal(p[lo:lo + 4096].cpu(), x[lo:lo + 4096].bfloat16())
    del ballast
    L.close()


def test_c_example_matches_the_oracle(lamb, tmp_path):
    """examples/lamb_c_example.c — the C ABI from plain C (no Python in the step path): its trust
    ratios and first master weights after two toy steps equal the oracle's."""
    import re
    import subprocess
    lib_dir = os.path.dirname(lamb.LIB_PATH)
    exe = str(tmp_path / "lamb_c_example")
    r = subprocess.run(["gcc", "-std=c11", "-O2", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "lamb_c_example.c"), "-o", exe, "-L", lib_dir, "-llamb",
                        f"-Wl,-rpath,{lib_dir}", "-lm"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    orc = oracle.OracleRun(W.toy(), world_size=1)
    orc.step(1)
    orc.step(2)
    ratios = [float(x) for x in re.findall(r"trust ratio = ([0-9.eE+-]+)", r.stdout)]
    assert len(ratios) == 3
    for i, got in enumerate(ratios):
        assert abs(got - orc.stats[i][2]) <= 1e-5 * abs(orc.stats[i][2]) + 1e-6, (i, got, orc.stats[i])
    w = [float(x) for x in re.search(r"w\[0\.\.3\] = (\S+) (\S+) (\S+) (\S+)", r.stdout).groups()]
    for k in range(4):   # printed with 8 decimals
        assert abs(w[k] - orc.w[0][k]) <= 1e-8 + 1e-5 * abs(orc.w[0][k]), (k, w[k], orc.w[0][k])
