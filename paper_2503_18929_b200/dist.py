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


class PartialAllreduce:
    """The loss partials' all-reduce running on a side stream: the backward never
    waits for it, because the gradient needs only the static N_global. ``wait()`` makes the
    caller's current stream wait for it and returns the global [L, N_global, B_global]."""

    def __init__(self, out, event, stream):
        self.out, self.event, self.stream = out, event, stream

    def wait(self):
        import torch
        torch.cuda.current_stream(self.out.device).wait_event(self.event)
        self.out.record_stream(torch.cuda.current_stream(self.out.device))
        return self.out


_SIDE: dict = {}


def allreduce_partial_async(partial, group) -> PartialAllreduce:
    """All-reduce (sum) a copy of ``partial`` (fp64 [3], on the current stream's device) on a side
    stream ordered after the current stream's work so far; the current stream does not wait. The
    result is read through ``PartialAllreduce.wait()`` (event-ordered)."""
    import torch
    import torch.distributed as dist
    dev = partial.device
    key = (dev.type, dev.index)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
    side = _SIDE[key]
    if side is None:  # CPU tensors (gloo tests): nothing to overlap
        out = partial.clone()
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
        return _CpuDone(out)
    cur = torch.cuda.current_stream(dev)
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        out = partial.clone()
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
        ev = torch.cuda.Event()
        ev.record(side)
    partial.record_stream(side)
    return PartialAllreduce(out, ev, side)


class _CpuDone:
    def __init__(self, out):
        self.out = out

    def wait(self):
        return self.out
