"""Comm-aware partitioner: exact against brute force on
the paper's RevNets, and it moves cuts away from the large early boundaries when
the link is slow."""
import itertools

import pytest

from paper_2406_02052_b200 import models as PM
from paper_2406_02052_b200.dist import contiguous_stage_ranks


def modelled(units, counts, world, H, link=PM.LINK_BPS):
    cost = PM.unit_cost(units, 64, H, H, 3)
    bnd = PM.boundary_bytes(units, 64, H, H, 3)
    ranks = contiguous_stage_ranks(len(counts), world)
    starts = [sum(counts[:j]) for j in range(len(counts))] + [len(units)]
    worst = 0.0
    for g in range(world):
        js = [j for j, r in enumerate(ranks) if r == g]
        i0, i1 = starts[js[0]], starts[js[-1] + 1]
        t = sum(cost[i0:i1]) + ((bnd[i0] if i0 > 0 else 0) + (bnd[i1] if i1 < len(units) else 0)) / link
        worst = max(worst, t)
    return worst


def brute(units, J, world, H):
    n = len(units)
    best = float("inf")
    for cuts in itertools.combinations(range(1, n), J - 1):
        b = (0,) + cuts + (n,)
        counts = [b[i + 1] - b[i] for i in range(J)]
        best = min(best, modelled(units, counts, world, H))
    return best


@pytest.mark.parametrize("model,H", [("revnet18", 32), ("revnet50", 224)])
@pytest.mark.parametrize("J,world", [(4, 4), (4, 2), (8, 8), (8, 4)])
def test_partition_comm_is_optimal(model, H, J, world):
    units = PM.revnet(model, H, 10)
    counts = PM.partition_comm(units, J, world, 64, H, H, 3)
    assert len(counts) == J and sum(counts) == len(units) and min(counts) >= 1
    got = modelled(units, counts, world, H)
    assert got <= brute(units, J, world, H) * (1 + 1e-12)


def test_slow_link_moves_cuts_to_small_boundaries(monkeypatch):
    units = PM.revnet("revnet50", 224, 10)
    bnd = PM.boundary_bytes(units, 64, 224, 224, 3)
    fast = PM.partition_comm(units, 4, 4, 64, 224, 224, 3)
    monkeypatch.setattr(PM, "LINK_BPS", 1e9)   # a very slow link: cut bytes dominate
    slow = PM.partition_comm(units, 4, 4, 64, 224, 224, 3)
    cut_bytes = lambda c: sum(bnd[sum(c[:j])] for j in range(1, len(c)))
    assert cut_bytes(slow) <= cut_bytes(fast)
    assert cut_bytes(slow) == min(cut_bytes(list(c)) for c in _all_counts(len(units), 4))


def _all_counts(n, J):
    for cuts in itertools.combinations(range(1, n), J - 1):
        b = (0,) + cuts + (n,)
        yield [b[i + 1] - b[i] for i in range(J)]
