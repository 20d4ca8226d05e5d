"""Whole-group sharding across ranks.

Eq. 4 couples only the K samples of one prompt, so prompt groups are independent: each
rank takes a contiguous block of whole groups, runs the head on it with the GLOBAL
normaliser n_seq_global = B_global * K (Eq. 5's 1/(BK)), and one all-reduce of
partial = [sum eps^2 / N_global, n_seq, n_groups] yields the loss. The backward needs no
collective (N_global is static).
"""
from __future__ import annotations


def group_range(n_groups: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced (sizes differ by at most 1) block of whole groups for `rank`."""
    if world < 1 or not (0 <= rank < world) or n_groups < 0:
        raise ValueError("bad world/rank/n_groups")
    base, rem = divmod(n_groups, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def token_balanced_ranges(group_tokens, world: int) -> list[tuple[int, int]]:
    """Contiguous whole-group blocks balancing the number of VALID rows per rank (for
    ragged masks, e.g. RhoMath's up-to-512-token responses): greedy prefix cut at the
    ideal per-rank share. Returns one [start, end) per rank (possibly empty)."""
    import itertools
    tot = sum(group_tokens)
    cum = list(itertools.accumulate(group_tokens))
    cuts, g = [0], 0
    for r in range(1, world):
        target = tot * r / world
        while g < len(cum) and cum[g] <= target:
            g += 1
        # pick the closer of cutting before/after group g
        if g < len(cum):
            before = cum[g - 1] if g > 0 else 0
            if abs(cum[g] - target) < abs(before - target):
                g += 1
        g = max(g, cuts[-1])
        cuts.append(min(g, len(group_tokens)))
    cuts.append(len(group_tokens))
    return [(cuts[i], cuts[i + 1]) for i in range(world)]
