"""Data parallelism over images + embedding handoff to the LLM-backend GPU (K10).

The reference partitions a request's images over image instances with ``split_by_tiles``
(policies.py:91-124), waits for every shard before prefill (engine.py:746-749) and models the
token transfer as a lognormal delay (engine.py:42-67, :563-579).  Here the partition is real —
one process per GPU, replicated weights, no collective on the data path — and the transfer is
an NCCL point-to-point send of each rank's packed [tokens, D_out] bf16 slice to the LLM-backend
rank (pull semantics of PAPER.md:654-660: the receiver posts the receives into a buffer whose
offsets it computes itself from the deterministic tile plan, so no size exchange is needed).

Sends and receives are issued on NCCL's own stream and only waited on when their buffer is
about to be reused, so the transfer of step i overlaps compute of step i+1.  A sender whose
packed output always lands in the same buffer (a replayed CUDA graph) calls ``release(buf)``
before the kernels that rewrite it: the compute stream then waits for every pending send still
reading that buffer (a stream wait, not a host sync).
"""

from __future__ import annotations

from collections import deque

import torch
import torch.distributed as dist

from .policies import split_by_cost, split_by_tiles


def partition_images(tiles: list[int], n_ranks: int, costs: list[float] | None = None) -> list[list[int]]:
    """Image indices per rank: reference split_by_tiles (parity mode) or cost-weighted LPT
    (performance mode).  Always returns exactly n_ranks lists (possibly empty)."""
    shards = split_by_cost(costs, n_ranks) if costs is not None else split_by_tiles(tiles, n_ranks)
    shards = shards + [[] for _ in range(n_ranks - len(shards))]
    return shards


class Handoff:
    """Per-step P2P handoff of packed embeddings from every rank to ``dst``."""

    def __init__(self, rank: int, world: int, dst: int = 0, depth: int = 2):
        self.rank, self.world, self.dst, self.depth = rank, world, dst, depth
        self.pending: deque = deque()
        self.received: list = []  # rank dst: the last step's received buffers, by source rank

    def _retire(self, keep: int):
        while len(self.pending) > keep:
            works, _bufs = self.pending.popleft()
            for w in works:
                w.wait()

    def release(self, buf: torch.Tensor):
        """Order the current stream after every pending send or receive that uses ``buf``'s
        memory (call before rewriting a buffer that was handed to ``send``)."""
        lo = buf.data_ptr()
        hi = lo + buf.numel() * buf.element_size()
        keep: deque = deque()
        for works, payload in self.pending:
            tensors = payload.values() if isinstance(payload, dict) else (payload,)
            if any(t.data_ptr() < hi and lo < t.data_ptr() + t.numel() * t.element_size() for t in tensors):
                for w in works:
                    w.wait()
            else:
                keep.append((works, payload))
        self.pending = keep

    def send(self, packed, sizes: dict | None = None, width: int | None = None):
        """packed: PackedBatch (or a tensor) of this rank.  On ``dst``, ``sizes`` maps source rank ->
        token rows to receive (default: same shape as the local tensor)."""
        emb = packed.embeds if hasattr(packed, "embeds") else packed
        self._retire(self.depth - 1)
        if self.rank == self.dst:
            ops, bufs = [], {}
            for src in range(self.world):
                if src == self.dst:
                    continue
                rows = sizes[src] if sizes else emb.shape[0]
                buf = torch.empty(rows, width or emb.shape[1], dtype=emb.dtype, device=emb.device)
                bufs[src] = buf
                ops.append(dist.P2POp(dist.irecv, buf, src))
            works = dist.batch_isend_irecv(ops) if ops else []
            self.received = bufs
            self.pending.append((works, bufs))
        else:
            works = dist.batch_isend_irecv([dist.P2POp(dist.isend, emb, self.dst)])
            self.pending.append((works, emb))

    def flush(self):
        self._retire(0)
