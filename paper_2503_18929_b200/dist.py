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


class PeerReducer:
    """Buffers for the loss all-reduce fused into the head kernel over peer memory
    (tba_tb_loss_fwd_peer; CUDA IPC mappings, P2P over NVLink). Collective: every rank of
    ``group`` constructs it once on its device; ``next_args()`` returns the per-call struct
    (the epoch increases by one per call on every rank)."""

    def __init__(self, group, device, timeout_s: float = 10.0):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib
        L = _lib.load()
        self._L = L
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.timeout_s = float(timeout_s)
        self.device = torch.device(device)
        own = []
        handles = []
        with torch.cuda.device(self.device):
            for nbytes in (2 * self.world * 4 * 8, max(self.world * 4, 16)):
                ptr = ctypes.c_void_p()
                h = ctypes.create_string_buffer(64)
                _lib.check(L.tba_ipc_alloc(nbytes, ctypes.byref(ptr), h), "tba_ipc_alloc")
                own.append(ptr.value)
                handles.append(h.raw)
        self._own = own
        gathered = [None] * self.world
        dist.all_gather_object(gathered, handles, group=group)
        self._opened = []
        slots, flags = [], []
        with torch.cuda.device(self.device):
            for q in range(self.world):
                if q == self.rank:
                    slots.append(own[0])
                    flags.append(own[1])
                    continue
                ptrs = []
                for h in gathered[q]:
                    p = ctypes.c_void_p()
                    _lib.check(L.tba_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)), "tba_ipc_open")
                    self._opened.append(p.value)
                    ptrs.append(p.value)
                slots.append(ptrs[0])
                flags.append(ptrs[1])
        # device arrays of device pointers
        self.slots_arr = torch.tensor(slots, dtype=torch.int64, device=self.device)
        self.flags_arr = torch.tensor(flags, dtype=torch.int64, device=self.device)
        self.epoch = 0
        dist.barrier(group=group)

    def next_args(self):
        from ._lib import TbaPeerReduce
        self.epoch += 1
        return TbaPeerReduce(self.slots_arr.data_ptr(), self.flags_arr.data_ptr(), self.rank, self.world,
                             self.epoch, self.timeout_s)

    def close(self):
        import torch
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            self._L.tba_ipc_close(p)
        for p in self._own:
            self._L.tba_ipc_free(p)
        self._opened, self._own = [], []
