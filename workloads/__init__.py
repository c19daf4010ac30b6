"""Seeded synthetic workloads (inputs only) shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no LAMB math, no planner rules).  It only
describes *inputs*: the parameter-tensor tables shaped like the paper's models, the
hyper-parameter groups, and the generator recipe's per-tensor parameters.  Both
`oracle/` (test infrastructure) and `paper_2402_15627_b200/` (the product) read it; each
side implements the Philox4x32-10 generator itself.

Shapes follow PAPER.md Table `tab:exp-model-config` (175B h=12288, 530B
h=20480), seq/vocab P:828-829 (vocab 64,000), and the GPT-style layer pattern of a
Megatron-LM transformer.  Per-config tensor counts/sizes are SURVEY.md §8(d).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

# init kinds for the fp32 master weights (SURVEY.md §8(d) "Weights")
INIT_UNIFORM = 0   # w = (int(x>>8) - 2^23) * 2^-28, uniform on [-1/32, 1/32)
INIT_ONE = 1       # LayerNorm weight
INIT_ZERO = 2      # biases, LayerNorm bias, even stress tensors

# generator streams (SURVEY.md §8(d) "Philox4x32-10")
STREAM_WEIGHTS = 1
STREAM_GRADS = 2

# gradient exponent base E (value = ±(1+mant/128)·2^(E-k), k∈{0..3})
GEXP_MATRIX = -10
GEXP_VECTOR = -8

BASE_SEED = 0x4D454741  # "MEGA"

# fp32 hyper-parameter values (readings Z4, Z6, Z7, Z13)
LR_BENCH = 2.0 ** -10
BETA1 = 0.9
BETA2 = 0.999
EPS = 1e-6
WD_DECAY = 0.01


@dataclass(frozen=True)
class TensorSpec:
    name: str
    numel: int
    group: int          # index into Workload.groups
    init: int           # INIT_*
    gexp: int           # GEXP_*


@dataclass(frozen=True)
class GroupSpec:
    lr: float = LR_BENCH
    beta1: float = BETA1
    beta2: float = BETA2
    eps: float = EPS
    weight_decay: float = 0.0
    adapt: int = 1
    bias_correction: int = 1


@dataclass
class Workload:
    name: str
    index: int                       # config index → seed = BASE_SEED + index
    tensors: List[TensorSpec]
    groups: List[GroupSpec]
    cap: int = 40_000_000            # bucket cap in elements (P3)
    world_sizes: tuple = (1,)
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index

    @property
    def n_params(self) -> int:
        return sum(t.numel for t in self.tensors)


DECAY, NO_DECAY = 0, 1


def default_groups(lr: float = LR_BENCH) -> List[GroupSpec]:
    return [GroupSpec(lr=lr, weight_decay=WD_DECAY),   # DECAY: >=2-D tensors incl. embedding
            GroupSpec(lr=lr, weight_decay=0.0)]        # NO_DECAY: 1-D tensors


def _mat(name, rows, cols):
    return TensorSpec(name, rows * cols, DECAY, INIT_UNIFORM, GEXP_MATRIX)


def _vec(name, n, init):
    return TensorSpec(name, n, NO_DECAY, init, GEXP_VECTOR)


def gpt_layer(prefix: str, h: int) -> List[TensorSpec]:
    """One GPT/Megatron transformer layer's parameter tensors, in table order."""
    return [
        _vec(f"{prefix}.ln1.w", h, INIT_ONE), _vec(f"{prefix}.ln1.b", h, INIT_ZERO),
        _mat(f"{prefix}.qkv.w", 3 * h, h), _vec(f"{prefix}.qkv.b", 3 * h, INIT_ZERO),
        _mat(f"{prefix}.proj.w", h, h), _vec(f"{prefix}.proj.b", h, INIT_ZERO),
        _vec(f"{prefix}.ln2.w", h, INIT_ONE), _vec(f"{prefix}.ln2.b", h, INIT_ZERO),
        _mat(f"{prefix}.fc1.w", 4 * h, h), _vec(f"{prefix}.fc1.b", 4 * h, INIT_ZERO),
        _mat(f"{prefix}.fc2.w", h, 4 * h), _vec(f"{prefix}.fc2.b", h, INIT_ZERO),
    ]


def gpt(h: int, layers: int, vocab: int | None = 64_000, final_ln: bool = True) -> List[TensorSpec]:
    ts: List[TensorSpec] = []
    if vocab:
        ts.append(_mat("emb", vocab, h))
    for i in range(layers):
        ts += gpt_layer(f"l{i}", h)
    if final_ln:
        ts += [_vec("lnf.w", h, INIT_ONE), _vec("lnf.b", h, INIT_ZERO)]
    return ts


def stress_tensors(k0: int, k1: int) -> List[TensorSpec]:
    """Segmented-norm stress set: numel 1 + (k*2654435761 mod 4099); even k start at 0."""
    out = []
    for k in range(k0, k1):
        n = 1 + (k * 2654435761) % 4099
        out.append(TensorSpec(f"s{k}", n, NO_DECAY, INIT_ZERO if k % 2 == 0 else INIT_UNIFORM,
                              GEXP_VECTOR))
    return out


def toy() -> Workload:
    # SURVEY.md §8(d) toy: t0 [64,48] decay; t1 [48] no_decay; t2 [128,64] decay.
    ts = [_mat("t0", 64, 48), _vec("t1", 48, INIT_ZERO), _mat("t2", 128, 64)]
    return Workload("toy", 0, ts, default_groups(), world_sizes=(1, 2))


def gpt_1p3b() -> Workload:
    return Workload("gpt1.3b", 1, gpt(2048, 24), default_groups(), world_sizes=(1, 2, 4, 8))


def gpt_13b() -> Workload:
    return Workload("gpt13b", 2, gpt(5120, 40), default_groups(), world_sizes=(2, 4, 8))


def slice_175b(layers: int = 12) -> Workload:
    name = "175b_slice" if layers == 12 else f"175b_slice_{layers}l"
    idx = 3 if layers == 12 else 5
    return Workload(name, idx, gpt(12288, layers, vocab=None, final_ln=False), default_groups(),
                    world_sizes=(4, 8) if layers == 12 else (1, 2, 4, 8))


def slice_530b_stress() -> Workload:
    ts: List[TensorSpec] = []
    for i in range(4):
        ts += gpt_layer(f"l{i}", 20480)
        ts += stress_tensors(8192 * i, 8192 * (i + 1))
    return Workload("530b_stress", 4, ts, default_groups(), cap=1_000_000, world_sizes=(4, 8))


CONFIGS = {
    "toy": toy,
    "gpt1.3b": gpt_1p3b,
    "gpt13b": gpt_13b,
    "175b_slice": lambda: slice_175b(12),
    "175b_slice_3l": lambda: slice_175b(3),
    "530b_stress": slice_530b_stress,
}


def get(name: str) -> Workload:
    return CONFIGS[name]()


def random_table(rng, n_tensors: int, max_numel: int = 5000, p_big: float = 0.1,
                 big: int = 40_000) -> List[TensorSpec]:
    """Ragged random table for parity edge cases (sizes 1.., some > small caps)."""
    out = []
    for i in range(n_tensors):
        if rng.random() < p_big:
            n = int(rng.integers(max_numel, big))
        else:
            n = int(rng.integers(1, max_numel))
        if rng.random() < 0.5:
            out.append(TensorSpec(f"r{i}", n, DECAY, INIT_UNIFORM, GEXP_MATRIX))
        else:
            init = [INIT_ONE, INIT_ZERO, INIT_UNIFORM][int(rng.integers(0, 3))]
            out.append(TensorSpec(f"r{i}", n, NO_DECAY, init, GEXP_VECTOR))
    return out
