"""Time-domain decomposition and the inter-rank transport.

Decomposition keeps the ownership rule of reference runtime.py:31-105
(whole C-intervals per rank, remainder to the lowest ranks, the last active
rank owns any F-tail, ranks beyond the interval count idle on that level),
tabulated as per-rank arrays.

The transport replaces the reference's queue-based p2p (runtime.py:123-254)
with torch.distributed: one process per GPU, NCCL over NVLink/NVSwitch for
device tensors (gloo for CPU tests).  Every exchange step of a sweep is one
grouped batch_isend_irecv (an ncclGroupStart/End), norms are an all-gather
of per-rank partial sums reduced in rank order on every rank (the
determinism of runtime.py:189-203), maxima an all-reduce.
"""

import numpy as np
import torch

from .errors import TransportError


class Decomposition:
    """Ownership of one level's C-intervals across n_workers ranks
    (semantics of reference runtime.py:31-105).

    Everything is tabulated once as arrays over ranks -- interval counts,
    first interval, owned point range [lo, hi) -- so the per-sweep queries of
    the engine are O(1) lookups and owner searches are binary searches:

        counts[w]  = K // p (+1 for the first K % p ranks)
        first[w]   = exclusive prefix sum of counts
        lo[w]      = C[first[w]] + 1,  hi[w] = C[first[w] + counts[w]] + 1
                     (the last rank that owns anything also owns the F-tail)

    Ranks past the interval count own nothing on this level; a level without
    any closed interval (fewer points than the factor) belongs to rank 0."""

    def __init__(self, splitting, n_workers):
        if n_workers < 1:
            raise ValueError(f"n_workers must be >= 1, got {n_workers}")
        self.splitting = splitting
        self.n_workers = int(n_workers)
        K, p = int(splitting.n_intervals), self.n_workers
        ranks = np.arange(p)
        self._counts = K // p + (ranks < K % p).astype(np.int64)
        self._first = np.concatenate(([0], np.cumsum(self._counts)[:-1])).astype(np.int64)
        self._ends = self._first + self._counts          # one past the last owned interval
        c = np.asarray(splitting.c_indices, dtype=np.int64)
        self._lo = np.zeros(p, dtype=np.int64)
        self._hi = np.zeros(p, dtype=np.int64)
        if K == 0:
            self._lo[0], self._hi[0] = 1, splitting.n_points
            self._idle = ranks > 0
        else:
            self._idle = self._counts == 0
            own = ~self._idle
            self._lo[own] = c[self._first[own]] + 1
            self._hi[own] = c[self._ends[own]] + 1
            self._hi[np.nonzero(own)[0][-1]] = splitting.n_points      # F-tail
        self._active = [int(w) for w in np.nonzero(~self._idle)[0]]

    def n_units(self, rank):
        return int(self._counts[rank])

    def first_unit(self, rank):
        return int(self._first[rank])

    def unit_owner(self, unit):
        if not 0 <= unit < self.splitting.n_intervals:
            raise ValueError(f"unit {unit} out of range")
        return int(np.searchsorted(self._ends, unit, side="right"))

    def is_empty(self, rank):
        return bool(self._idle[rank])

    def c_points(self, rank):
        f = int(self._first[rank])
        return self.splitting.c_indices[f + 1: f + 1 + int(self._counts[rank])]

    def left_boundary_index(self, rank):
        return int(self.splitting.c_indices[self._first[rank]])

    def owned_range(self, rank):
        return (int(self._lo[rank]), int(self._hi[rank]))

    def point_owner(self, point):
        """Rank whose owned range contains point (index 0 -> rank 0)."""
        if point == 0:
            return 0
        act = self._active
        k = int(np.searchsorted(self._hi[act], point, side="right"))
        if k < len(act) and self._lo[act[k]] <= point:
            return act[k]
        raise RuntimeError(f"point {point} has no owner")

    def active_ranks(self):
        return list(self._active)

    def left_neighbor(self, rank):
        below = [w for w in self._active if w < rank]
        return below[-1] if below else None

    def right_neighbor(self, rank):
        above = [w for w in self._active if w > rank]
        return above[0] if above else None


class _Done:
    """Handle of an exchange that has nothing left to wait for."""

    def wait(self):
        pass


class _Pending:
    """In-flight grouped p2p batch.  wait() orders the caller's stream after
    the transfers (NCCL: a stream dependency, the host does not block) and
    lands host-staged receives in their device buffers (gloo)."""

    def __init__(self, reqs, staged):
        self.reqs, self.staged = reqs, staged

    def wait(self):
        for req in self.reqs:
            req.wait()
        for _, h, t in self.staged:
            t.copy_(h)
        self.reqs, self.staged = [], []


class NullTransport:
    """Single worker: no peers (reference runtime.py:110-120)."""

    rank = 0
    size = 1

    def exchange(self, sends, recvs):
        if sends or recvs:
            raise TransportError("no peers in a single-worker run")

    def exchange_async(self, sends, recvs):
        self.exchange(sends, recvs)
        return _Done()

    def sum_ordered(self, value):
        return float(value)

    def max(self, value):
        return float(value)

    def barrier(self):
        pass


class DistTransport:
    """torch.distributed transport (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise TransportError("torch.distributed is not initialised")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cpu")
        # gloo moves host tensors only: device buffers are staged through the
        # host (tests run several ranks on one GPU this way); NCCL moves device
        # tensors directly over NVLink
        self.stage = dist.get_backend(group) != "nccl" and self.device.type == "cuda"
        cdev = torch.device("cpu") if self.stage else self.device
        self.coll_device = cdev
        # the first collective must involve every rank (NCCL p2p rule)
        t = torch.zeros(1, dtype=torch.float64, device=cdev)
        dist.all_reduce(t, group=group)

    def exchange(self, sends, recvs):
        """sends/recvs: lists of (peer, tensor); one grouped p2p batch."""
        self.exchange_async(sends, recvs).wait()

    def exchange_async(self, sends, recvs):
        """Start the grouped p2p batch and return a handle; the transfers run
        on the communicator's stream (NCCL over NVLink) while the caller keeps
        issuing work that does not touch the receive buffers, then wait()."""
        if self.stage:
            sends = [(peer, t.detach().to("cpu")) for peer, t in sends]
            staged = [(peer, torch.empty(t.shape, dtype=t.dtype), t) for peer, t in recvs]
            recvs_h = [(peer, h) for peer, h, _ in staged]
        else:
            recvs_h, staged = recvs, []
        ops = [self.dist.P2POp(self.dist.isend, t.contiguous(), peer, self.group)
               for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, self.group)
                for peer, t in recvs_h]
        if not ops:
            return _Done()
        return _Pending(self.dist.batch_isend_irecv(ops), staged)

    def sum_ordered(self, value):
        """Rank-ascending sum of per-rank partials, identical on every rank."""
        t = torch.tensor([float(value)], dtype=torch.float64, device=self.coll_device)
        out = [torch.zeros_like(t) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        vals = torch.cat(out).cpu().numpy()
        total = 0.0
        for v in vals:
            total += float(v)
        return total

    def max(self, value):
        t = torch.tensor([float(value)], dtype=torch.float64, device=self.coll_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)


def plan_moves(points, src_owner, dst_owner, rank):
    """Route per-point rows from producer to consumer ranks.

    points: increasing global point indices; src_owner / dst_owner: owner
    rank per point (every rank computes the same arrays).  Returns
    (local, sends, recvs), each a list of (peer, lo, hi) runs of
    consecutive points with one (src, dst) pair."""
    points = np.asarray(points)
    src_owner = np.asarray(src_owner)
    dst_owner = np.asarray(dst_owner)
    local, sends, recvs = [], [], []
    i, n = 0, len(points)
    while i < n:
        j = i + 1
        while (j < n and src_owner[j] == src_owner[i] and dst_owner[j] == dst_owner[i]
               and points[j] == points[j - 1] + 1):
            j += 1
        s, d = int(src_owner[i]), int(dst_owner[i])
        run = (int(points[i]), int(points[j - 1]) + 1)
        if s == rank and d == rank:
            local.append((rank,) + run)
        elif s == rank:
            sends.append((d,) + run)
        elif d == rank:
            recvs.append((s,) + run)
        i = j
    return local, sends, recvs
