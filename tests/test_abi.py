"""CPU checks of the boundary: liblamb.so loads without a GPU, exports every symbol the
headers declare, and its host planner (row a0) equals the oracle planner bit-exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import workloads as W
from paper_2402_15627_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    from paper_2402_15627_b200 import lamb
    return lamb


def declared_functions():
    names = []
    for h in ("lamb.h", "lamb_synth.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s+(lamb_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 20
    so = ctypes.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(so, n), n
    assert set(names) == set(L.exported_symbols())


def test_errors_without_gpu_are_reported(L):
    # argument validation happens before any device call
    v = L.lamb_group(1e-3, 0.9, 1.5, 1e-6, 0.0, 1, 1)   # beta2 out of range
    t = (L.lamb_tensor * 1)(L.lamb_tensor(10, 0, 0))
    cfg = L.lamb_config(1, 0, 0, 1, 0, 0.0, 0)
    h = ctypes.c_void_p()
    st = L.lamb_create(t, 1, (L.lamb_group * 1)(v), 1, ctypes.byref(cfg), None, ctypes.byref(h))
    assert st == L.LAMB_EINVAL and b"beta2" in L.lamb_last_error(None)
    with pytest.raises(L.LambError):
        L.host_plan([5, 0], 1, 0)
    h0 = ctypes.c_void_p()
    assert L.lamb_plan_create(t, 0, 1, 0, 0, ctypes.byref(h0)) == L.LAMB_EINVAL   # empty table
    with pytest.raises(L.LambError):
        L.host_plan([5], 9, 0)
    with pytest.raises(L.LambError):
        L.host_plan([5], 2, 2)


def test_binding_rejects_mis_sized_host_buffers(L):
    # the C side reads flat_size elements from the pointer it is given: the binding checks
    # size, dtype and layout before handing a tensor over
    import torch
    n = 1024
    L._check_flat(torch.zeros(n, dtype=torch.bfloat16), n, L._BF16_LIKE, "g", cuda=False)
    L._check_flat(torch.zeros(n, dtype=torch.int16), n, L._BF16_LIKE, "g", cuda=False)
    with pytest.raises(ValueError, match="elements"):
        L._check_flat(torch.zeros(n - 8, dtype=torch.bfloat16), n, L._BF16_LIKE, "g")
    with pytest.raises(ValueError, match="dtype"):
        L._check_flat(torch.zeros(n, dtype=torch.float32), n, L._BF16_LIKE, "g")
    with pytest.raises(ValueError, match="dtype"):
        L._check_flat(torch.zeros(n, dtype=torch.float64), n, ("torch.float32",), "w")
    with pytest.raises(ValueError, match="contiguous"):
        L._check_flat(torch.zeros(2 * n, dtype=torch.bfloat16)[::2], n, L._BF16_LIKE, "g")
    with pytest.raises(ValueError, match="CUDA"):
        L._check_flat(torch.zeros(n, dtype=torch.bfloat16), n, L._BF16_LIKE, "g", cuda=True)


def compare(L, numels, D, cap):
    op = oracle.plan(numels, D, cap)
    for r in range(D):
        lp = L.host_plan(numels, D, r, cap)
        assert lp.flat_size == op.flat_size and lp.shard_size == op.shard_size
        assert lp.tensor_off.tolist() == op.tensor_off
        assert lp.tensor_bucket.tolist() == op.tensor_bucket
        assert [tuple(b) for b in lp.buckets.tolist()] == op.buckets
        assert [tuple(s) for s in lp.segments.tolist()] == op.segments[r]
        assert lp.straddlers.tolist() == op.straddlers


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_planner_bit_exact_vs_oracle(L, name):
    wl = W.get(name)
    numels = [t.numel for t in wl.tensors]
    Ds = (1, 2, 4, 8) if name != "530b_stress" else (8,)
    for D in Ds:
        compare(L, numels, D, wl.cap)


@pytest.mark.parametrize("seed", range(8))
def test_planner_bit_exact_random(L, seed):
    rng = np.random.default_rng(1000 + seed)
    numels = [t.numel for t in W.random_table(rng, int(rng.integers(1, 80)), max_numel=5000,
                                              p_big=0.1, big=50000)]
    cap = int(rng.choice([0, 1, 64, 1000, 8192, 30000]))
    for D in range(1, 9):
        compare(L, numels, D, cap if cap else 40_000_000)


def test_binding_fails_loudly_without_the_library(tmp_path):
    # no CPU fallback: a copy of the binding next to no liblamb.so refuses to import
    import importlib.util
    import shutil
    src = os.path.join(ROOT, "paper_2402_15627_b200", "lamb.py")
    dst = tmp_path / "lamb_copy.py"
    shutil.copy(src, dst)
    spec = importlib.util.spec_from_file_location("lamb_copy", dst)
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError, match="no CPU fallback"):
        spec.loader.exec_module(mod)


def test_debug_build_exports_its_hooks_and_carries_the_checks(L):
    # liblamb_debug.so (-DLAMB_DEBUG): the release ABI plus lamb_debug.h's hook, and device-side
    # checks (trap sites) that the release library does not contain
    import subprocess
    dbg = B.build(debug=True)
    so = ctypes.CDLL(dbg)
    for n in declared_functions():
        assert hasattr(so, n), n
    assert hasattr(so, "lamb_debug_corrupt_item")
    assert not hasattr(ctypes.CDLL(B.build()), "lamb_debug_corrupt_item")

    def traps(path):
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        return sass.count("BPT.TRAP")
    assert traps(dbg) > 50 and traps(B.build()) == 0


def _compile_c_example(L, out):
    import subprocess
    lib_dir = os.path.dirname(L.LIB_PATH if not L.DEBUG else B.build())
    return subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "lamb_c_example.c"), "-o", out, "-L", lib_dir, "-llamb",
                           f"-Wl,-rpath,{lib_dir}", "-lm"], capture_output=True, text=True)


def test_c_example_compiles_against_the_headers(L, tmp_path):
    # the boundary is plain C: the example builds with gcc against include/*.h and liblamb.so alone
    r = _compile_c_example(L, str(tmp_path / "lamb_c_example"))
    assert r.returncode == 0, r.stderr
