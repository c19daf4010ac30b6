"""Host logic of LambOptimizer(overlap=True) on CPU (no GPU): the BucketOverlap bookkeeping that
decides when the copy-engine schedule pushes a bucket's gradients (once per bucket per step, as
soon as the backward has accumulated its last parameter — PAPER.md §3.2: RS right
after a chunk's backward) and when the next forward waits for a bucket's all-gather (once, right
before the first module using it — P:319-327).  The GPU calls are replaced by recorders."""
import pytest

torch = pytest.importorskip("torch")

from paper_2402_15627_b200.torch_optim import BucketOverlap  # noqa: E402


class Rec:
    def __init__(self):
        self.pushes, self.waits = [], []

    def push(self, b, t):
        self.pushes.append((b, t))

    def wait(self, b, t):
        self.waits.append((b, t))


def _model():
    torch.manual_seed(0)
    return torch.nn.ModuleDict({
        "l1": torch.nn.Linear(4, 8),      # params 0, 1 -> bucket 0
        "l2": torch.nn.Linear(8, 3),      # params 2, 3 -> buckets 1, 2
        "unused": torch.nn.Linear(3, 3),  # params 4, 5 -> bucket 3 (never in the forward)
    })


def _fwd(m, x):
    return m["l2"](torch.relu(m["l1"](x))).sum()


def test_push_once_per_bucket_in_backward_order_and_wait_once_per_bucket_in_forward():
    m = _model()
    params = list(m.parameters())
    bucket_of = [0, 0, 1, 2, 3, 3]
    r = Rec()
    ov = BucketOverlap(params, bucket_of, 4, push=r.push, wait=r.wait)
    hooks = ov.install()
    try:
        x = torch.randn(5, 4)
        # step 1: no staged step yet -> no waits; the backward pushes buckets 1, 2 before 0
        _fwd(m, x).backward()
        assert r.waits == []
        assert sorted(r.pushes) == [(0, 1), (1, 1), (2, 1)]
        assert r.pushes[-1] == (0, 1)                      # l1 is the last in backward order
        ov.before_step(1)                                  # the unused bucket still gets pushed
        assert r.pushes[-1] == (3, 1) and len(r.pushes) == 4
        ov.after_step(1)
        # step 2: every used bucket awaited once, in forward order, before its module runs
        for p in params:
            p.grad = None
        loss = _fwd(m, x)
        assert r.waits == [(0, 1), (1, 1), (2, 1)]
        loss.backward()
        assert sorted(r.pushes[4:]) == [(0, 2), (1, 2), (2, 2)]
        ov.before_step(2)                                  # waits for the bucket no module used
        assert r.waits[-1] == (3, 1) and len(r.waits) == 4
        assert r.pushes[-1] == (3, 2) and len(r.pushes) == 8
        ov.after_step(2)
        _fwd(m, x)
        assert r.waits[4:] == [(0, 2), (1, 2), (2, 2)]
    finally:
        for h in hooks:
            h.remove()


def test_hooks_removed_leave_other_models_alone():
    m = _model()
    params = list(m.parameters())
    r = Rec()
    ov = BucketOverlap(params, [0] * len(params), 1, push=r.push, wait=r.wait)
    hooks = ov.install()
    ov.after_step(1)
    other = torch.nn.Linear(4, 2)
    other(torch.randn(3, 4)).sum().backward()   # not ours: no wait, no push
    assert r.waits == [] and r.pushes == []
    for h in hooks:
        h.remove()
    _fwd(m, torch.randn(2, 4)).backward()       # removed: nothing recorded
    assert r.waits == [] and r.pushes == []


def test_gradient_accumulation_pushes_only_the_last_micro_batch():
    """under gradient accumulation the buckets must be pushed once, by the last
    micro-batch's backward (no_sync() on the others); a second backward outside no_sync()
    before step() raises instead of letting the peers reduce a partial gradient."""
    m = _model()
    params = list(m.parameters())
    r = Rec()
    ov = BucketOverlap(params, [0, 0, 1, 2, 3, 3], 4, push=r.push, wait=r.wait)
    hooks = ov.install()
    try:
        x = torch.randn(5, 4)
        ov.sync = False                      # what LambOptimizer.no_sync() does
        _fwd(m, x).backward()
        _fwd(m, x).backward()
        assert r.pushes == []
        ov.sync = True
        _fwd(m, x).backward()                # the last micro-batch pushes every used bucket
        assert sorted(r.pushes) == [(0, 1), (1, 1), (2, 1)]
        with pytest.raises(RuntimeError, match="no_sync"):
            _fwd(m, x).backward()            # one more backward before step(): refused
        ov.before_step(1)
        ov.after_step(1)
        for p in params:
            p.grad = None
        _fwd(m, x).backward()                # the next step works normally again
        assert sorted(r.pushes[4:]) == [(0, 2), (1, 2), (2, 2)]
    finally:
        for h in hooks:
            h.remove()
