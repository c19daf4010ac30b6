"""Property-based check (hypothesis) that the library's C++ planner and the oracle's Python
planner (independent implementations of rules P1-P7) agree table-for-table on arbitrary
tables, world sizes and caps, including degenerate ones (1-element tensors, caps smaller than
every tensor, a single tensor)."""
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
from paper_2402_15627_b200 import build as B

B.build()
from paper_2402_15627_b200 import lamb  # noqa: E402

numels = st.lists(st.one_of(st.integers(1, 16), st.integers(1, 5000), st.integers(5000, 200_000)),
                  min_size=1, max_size=40)


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(numels=numels, D=st.integers(1, 8), cap=st.one_of(st.just(1), st.integers(8, 300_000)))
def test_library_planner_equals_oracle_planner(numels, D, cap):
    op = oracle.plan(numels, D, cap)
    for r in range(D):
        lp = lamb.host_plan(numels, D, r, cap)
        assert lp.flat_size == op.flat_size
        assert lp.tensor_off.tolist() == op.tensor_off
        assert [tuple(b) for b in lp.buckets.tolist()] == op.buckets
        assert [tuple(s) for s in lp.segments.tolist()] == op.segments[r]
        assert lp.straddlers.tolist() == op.straddlers
    # segments of all ranks tile every tensor exactly once
    cover = {}
    for r in range(D):
        for (i, soff, toff, ln) in op.segments[r]:
            cover.setdefault(i, []).append((toff, ln))
    for i, n in enumerate(numels):
        parts = sorted(cover[i])
        assert parts[0][0] == 0 and sum(l for _, l in parts) == n
