"""Oracle shard/bucket planner (rules P1-P7) in plain Python.  TEST INFRASTRUCTURE ONLY.

PAPER.md never mentions buckets or shard layouts; it only says ZeRO-2 shards optimizer
state and gradients across DP ranks (§2) and overlaps on a model-chunk basis
(§3.2).  The layout rules are DESIGN.md reading Z17 (= SURVEY.md §8(a) P1-P7),
the bit-exact contract between this planner and the library's C++ planner
(paper_2402_15627_b200/csrc/planner.cpp), which share no code.

P1 flat order = table order.
P2 each tensor start within its bucket rounded up to A_t = 8 elements.
P3 greedy close-before-overflow: for aligned size a, if the bucket is non-empty and
   size + a > cap, close it; then add the tensor.  Tensors never split across buckets.
P4 S_b = roundup(size_b, Q), Q = 128 * lcm(D, 8).
P5 base_b = sum of earlier S_b.
P6 rank r owns [base_b + r S_b/D, base_b + (r+1) S_b/D) of every bucket; shard-local
   order = bucket order.
P7 segment = tensor ∩ owned slice when non-empty; straddler = tensor with >= 2 segments.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import gcd
from typing import List, Tuple

A_T = 8      # tensor start alignment (elements)
A_S = 128    # slice granularity (elements)


def _roundup(x: int, q: int) -> int:
    return (x + q - 1) // q * q


@dataclass
class OraclePlan:
    world_size: int
    tensor_off: List[int]                  # flat offset of every tensor
    tensor_bucket: List[int]
    buckets: List[Tuple[int, int, int, int]]   # (base, S_b, t_begin, t_end)
    flat_size: int
    # per rank: list of segments (tensor, shard_off, tensor_off, len)
    segments: List[List[Tuple[int, int, int, int]]]
    shard_size: int                        # elements per rank (= flat_size / D)
    straddlers: List[int]                  # tensors with >= 2 segments, ascending


def plan(numels: List[int], world_size: int, cap: int = 40_000_000) -> OraclePlan:
    D = world_size
    assert D >= 1 and cap >= 1 and all(n >= 1 for n in numels)
    # P1-P3: bucket assignment and tensor starts within buckets
    bucket_members: List[List[int]] = []
    starts_in_bucket: List[int] = []
    size = 0
    for i, n in enumerate(numels):
        a = _roundup(n, A_T)
        if bucket_members and bucket_members[-1] and size + a > cap:
            size = 0
            bucket_members.append([])
        if not bucket_members:
            bucket_members.append([])
        starts_in_bucket.append(size)
        bucket_members[-1].append(i)
        size += a
    # P4-P5
    Q = A_S * (D * A_T // gcd(D, A_T))
    tensor_off = [0] * len(numels)
    tensor_bucket = [0] * len(numels)
    buckets = []
    base = 0
    for b, members in enumerate(bucket_members):
        last = members[-1]
        size_b = starts_in_bucket[last] + _roundup(numels[last], A_T)
        S_b = _roundup(size_b, Q)
        for i in members:
            tensor_off[i] = base + starts_in_bucket[i]
            tensor_bucket[i] = b
        buckets.append((base, S_b, members[0], members[-1] + 1))
        base += S_b
    flat = base
    # P6-P7
    segments: List[List[Tuple[int, int, int, int]]] = []
    count = [0] * len(numels)
    for r in range(D):
        segs = []
        shard_base = 0
        for (bbase, S_b, t0, t1) in buckets:
            sl = S_b // D
            lo, hi = bbase + r * sl, bbase + (r + 1) * sl
            for i in range(t0, t1):
                a, z = tensor_off[i], tensor_off[i] + numels[i]
                s, e = max(a, lo), min(z, hi)
                if s < e:
                    segs.append((i, shard_base + (s - lo), s - a, e - s))
                    count[i] += 1
            shard_base += sl
        segments.append(segs)
    straddlers = [i for i, c in enumerate(count) if c >= 2]
    return OraclePlan(D, tensor_off, tensor_bucket, buckets, flat, segments, flat // D, straddlers)
