"""Pins of the oracle planner (rules P1-P7, reading Z17): the worked example of
SURVEY.md Appendix A, structural invariants (H12) and the bucket/straddler counts that
SURVEY.md §8(a)/(d) lists for the BASELINE configs (computed in the survey session,
independently of this code)."""
import json
import os
from math import gcd

import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_appendix_a_worked_example():
    gold = json.load(open(os.path.join(GOLD, "planner_toy.json")))
    for D in (1, 2):
        pl = oracle.plan(gold["numel"], D, gold["cap"])
        assert pl.tensor_off == gold["tensor_off"]
        assert [list(b) for b in pl.buckets] == gold["buckets"]
        assert pl.flat_size == gold["flat_size"]
        assert [[list(s) for s in segs] for segs in pl.segments] == gold[f"D{D}"]["segments"]
        assert pl.straddlers == gold[f"D{D}"]["straddlers"]


def check_invariants(numels, D, cap):
    pl = oracle.plan(numels, D, cap)
    Q = 128 * (D * 8 // gcd(D, 8))
    # buckets tile the flat space
    base = 0
    for (b0, S, t0, t1) in pl.buckets:
        assert b0 == base and S % Q == 0 and S > 0 and t1 > t0
        base += S
        size = sum(((numels[i] + 7) // 8) * 8 for i in range(t0, t1))
        assert S - size < Q                       # minimal padding
        if t1 - t0 > 1:
            assert size <= cap                    # only a lone tensor may exceed cap
    assert base == pl.flat_size and pl.flat_size % D == 0
    # tensors: 8-aligned, in order, non-overlapping, inside their bucket
    prev_end = 0
    for i, n in enumerate(numels):
        o = pl.tensor_off[i]
        b0, S, t0, t1 = pl.buckets[pl.tensor_bucket[i]]
        assert o % 8 == 0 and o >= prev_end and b0 <= o and o + n <= b0 + S and t0 <= i < t1
        prev_end = o + n
    # close-before-overflow (strict >): the first tensor of every later bucket would have overflowed
    for b in range(1, len(pl.buckets)):
        _, _, t0p, t1p = pl.buckets[b - 1]
        size = sum(((numels[i] + 7) // 8) * 8 for i in range(t0p, t1p))
        a = ((numels[pl.buckets[b][2]] + 7) // 8) * 8
        assert size + a > cap
    # segments: cover every tensor exactly once, slices are multiples of 128
    cover = {}
    for r in range(D):
        shard = 0
        for (i, soff, toff, ln) in pl.segments[r]:
            b0, S, _, _ = pl.buckets[pl.tensor_bucket[i]]
            sl = S // D
            assert sl % 128 == 0
            flat = pl.tensor_off[i] + toff
            assert b0 + r * sl <= flat and flat + ln <= b0 + (r + 1) * sl
            cover.setdefault(i, []).append((toff, ln))
            assert soff >= shard
            shard = soff + ln
        assert shard <= pl.shard_size
    for i, n in enumerate(numels):
        parts = sorted(cover[i])
        pos = 0
        for toff, ln in parts:
            assert toff == pos
            pos += ln
        assert pos == n
    assert pl.straddlers == sorted(i for i, p in cover.items() if len(p) >= 2)
    return pl


@pytest.mark.parametrize("name", ["toy", "gpt1.3b", "gpt13b", "175b_slice", "175b_slice_3l"])
def test_H12_invariants_and_D_independence(name):
    wl = W.get(name)
    numels = [t.numel for t in wl.tensors]
    flats = set()
    for D in (1, 2, 4, 8):
        pl = check_invariants(numels, D, wl.cap)
        flats.add((tuple(pl.tensor_off), pl.flat_size))
    assert len(flats) == 1        # flat layout independent of D for D | 8 (P4)


def test_survey_bucket_counts():
    exp = {"toy": 1, "gpt1.3b": 37, "gpt13b": 242, "175b_slice": 97, "175b_slice_3l": 25,
           "530b_stress": 97}
    for name, nb in exp.items():
        wl = W.get(name)
        pl = oracle.plan([t.numel for t in wl.tensors], 8, wl.cap)
        assert len(pl.buckets) == nb, name


def test_survey_530b_stress_straddlers():
    wl = W.get("530b_stress")
    numels = [t.numel for t in wl.tensors]
    pl = check_invariants(numels, 8, wl.cap)
    small = [i for i in pl.straddlers if wl.tensors[i].name.startswith("s")]
    assert len(small) == 474
    assert len(pl.straddlers) == 474 + 38
    pl40 = oracle.plan(numels, 8, 40_000_000)
    assert len([i for i in pl40.straddlers if wl.tensors[i].name.startswith("s")]) == 28
    assert max(len(s) for s in pl.segments) <= 4219


@pytest.mark.parametrize("seed", range(6))
def test_H12_random_tables(seed):
    import numpy as np
    rng = np.random.default_rng(100 + seed)
    numels = [t.numel for t in W.random_table(rng, int(rng.integers(1, 60)), max_numel=3000,
                                              p_big=0.15, big=20000)]
    cap = int(rng.choice([1, 8, 1000, 4096, 10_000, 40_000_000]))
    for D in range(1, 9):
        check_invariants(numels, D, cap)


def test_exact_cap_tie_break():
    # a tensor that makes the bucket exactly `cap` joins it; the next one closes it (Z17)
    pl = oracle.plan([8, 8, 8], 1, cap=16)
    assert [(b[2], b[3]) for b in pl.buckets] == [(0, 2), (2, 3)]
    pl = oracle.plan([100, 5], 1, cap=50)    # oversized tensor gets its own bucket
    assert [(b[2], b[3]) for b in pl.buckets] == [(0, 1), (1, 2)]
