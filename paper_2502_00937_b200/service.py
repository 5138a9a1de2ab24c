"""Real-time image-path service: request replay through the modality-aware batcher.

The reference simulates this loop (engine.py:517-752): an arriving multimodal request is routed
to image instances (`route_image`, policies.py:104-124, least-pending over pending image tokens),
each instance forms batches from its queue (`form_batch`, engine.py:100-114), and prefill waits
for every shard (engine.py:746-749) after a transfer delay (engine.py:563-579).  Here it runs
for real: one process per GPU is one image instance, batches execute on the B200
(`ImagePathExecutor.run`), and each finished shard's packed embeddings are streamed to the
LLM-backend rank (rank 0), which joins the shards of every request.

Routing needs a consistent view of every instance's pending image tokens on all ranks without a
control-plane round trip, so each rank runs the same deterministic model of the instances
(FIFO servers whose service time comes from a latency profile, exactly as the reference's
simulator tracks `pending_image_tokens`) and computes the same assignment.

Latency of a request = time from its (replayed) arrival until the embeddings of all its images
are resident on rank 0.  Percentiles use the reference's nearest-rank rule (metrics.py:12-18).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import policies as pol
from .batcher import WorkItem, form_batch
from .core import ModelSpec, Request, StageKind


def quantile(values, q: float) -> float:
    """Nearest-rank (lower) quantile, the reference's definition (metrics.py:12-18)."""
    if not len(values):
        raise ValueError("quantile of empty data")
    ordered = sorted(values)
    return ordered[max(0, math.ceil(q * len(ordered)) - 1)]


@dataclass
class _InstanceModel:
    id: int
    pending_image_tokens: int = 0
    busy_until: float = 0.0
    inflight: list = field(default_factory=list)  # (finish_ms, tokens)

    def advance(self, now: float) -> None:
        keep = []
        for finish, tok in self.inflight:
            if finish <= now:
                self.pending_image_tokens -= tok
            else:
                keep.append((finish, tok))
        self.inflight = keep


def route_requests(requests: list[Request], n_instances: int, cost_ms, policies: pol.PolicySet | None = None):
    """Deterministic routing of every multimodal request over ``n_instances`` image instances.

    Returns {request id: [(instance, [image indices])]}.  ``cost_ms(tiles)`` is the modelled
    service time of a shard; pending tokens drain at the modelled finish times."""
    policies = policies or pol.PolicySet()
    insts = [_InstanceModel(k) for k in range(n_instances)]
    rr: dict = {}
    out = {}
    for r in sorted(requests, key=lambda r: (r.arrival_ms, r.id)):
        if not r.is_multimodal:
            continue
        for inst in insts:
            inst.advance(r.arrival_ms)
        res = pol.route_image(r, insts, policies.router, policies.max_fanout, rr)
        out[r.id] = [(inst.id, list(idx)) for inst, idx in res]
        for inst, idx in res:
            tiles = sum(r.images[i].tiles for i in idx)
            tok = sum(r.images[i].image_tokens for i in idx)
            start = max(r.arrival_ms, inst.busy_until)
            inst.busy_until = start + cost_ms(tiles)
            inst.pending_image_tokens += tok
            inst.inflight.append((inst.busy_until, tok))
    return out


def synthetic_image(req_id: int, idx: int, w: int, h: int) -> np.ndarray:
    rng = np.random.default_rng((req_id << 8) + idx)
    return rng.integers(0, 256, (h, w, 3), dtype=np.uint8)


class ShardChannel:
    """Streamed handoff of variable-size shard embeddings to rank 0.

    Each shard is a small int64 header (request id, shard id, rows, width) on a CPU (gloo)
    control group followed by the payload on the data group (NCCL between GPUs).  On rank 0 one
    receiver thread per source posts the receives and hands completed shards to the replay loop
    through a queue, so sources may finish shards in any order (real-time batching).  A header
    with request id -1 ends a source's stream."""

    @staticmethod
    def make_groups(world: int, backend_data: str | None = None):
        """Dedicated two-rank groups per source (control on gloo, data on the default backend):
        point-to-point traffic of different sources never serialises on a shared group.  Every
        rank must call this (group creation is collective)."""
        import torch.distributed as dist
        ctrl = {src: dist.new_group([0, src], backend="gloo") for src in range(1, world)}
        data = {src: dist.new_group([0, src], backend=backend_data) for src in range(1, world)}
        return ctrl, data

    def __init__(self, rank: int, world: int, device, dtype, ctrl_group=None, data_group=None, on_arrival=None,
                 on_receive=None):
        import queue
        import threading

        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.device, self.dtype = rank, world, device, dtype
        self.ctrl, self.data = ctrl_group, data_group
        self.on_arrival = on_arrival  # runs in the receiver thread, on its private stream
        self.on_receive = on_receive  # (request id, shard id, rows) hook before on_arrival (checks)
        self.outgoing = []
        self.ready = queue.Queue()
        self.ended = 0
        self.counts = {"peer": 0, "nccl": 0}  # rank 0: shards received per payload path
        self.threads = []
        if rank == 0:
            for src in range(1, world):
                th = threading.Thread(target=self._recv_loop, args=(src,), daemon=True)
                th.start()
                self.threads.append(th)

    def _recv_loop(self, src):
        torch, dist = self.torch, self.dist
        if self.device.type == "cuda":
            # receives are ordered on a private stream: an NCCL op waits for the *current* stream,
            # which must not be the stream the replay loop keeps busy with encode batches
            torch.cuda.set_device(self.device)
            torch.cuda.set_stream(torch.cuda.Stream(self.device))
        while True:
            hdr = torch.empty(self.HDR, dtype=torch.int64)
            dist.recv(hdr, src, group=self._g(self.ctrl, src))
            rid, sid, rows, width, slot, row0, last, _ = (int(v) for v in hdr.tolist())
            if rid < 0:
                self.ready.put(None)
                return
            if slot >= 0:  # payload already in this GPU's memory (PeerShardChannel)
                self.counts["peer"] += 1
                self._peer_arrival(src, rid, sid, rows, width, slot, row0, last)
                continue
            self.counts["nccl"] += 1
            buf = torch.empty(rows, width, dtype=self.dtype, device=self.device)
            work = dist.irecv(buf, src, group=self._g(self.data, src))
            if self.device.type == "cuda":
                import time as _t
                while not work.is_completed():  # NCCL: completion of the receive on the GPU
                    _t.sleep(0.0005)  # coarse poll: keeps the GIL free for the replay loop
            else:
                work.wait()
            if self.on_receive is not None:
                self.on_receive(rid, sid, buf)
            extra = self.on_arrival(buf) if self.on_arrival is not None else None
            if self.device.type == "cuda":
                buf.record_stream(torch.cuda.default_stream(self.device))  # consumed by the replay loop
            self.ready.put((rid, sid, buf if extra is None else extra))

    HDR = 8  # request id, shard id, rows, width, peer slot (-1: NCCL payload follows), first row, last, 0

    def _peer_arrival(self, *args):
        raise RuntimeError("peer-slot header on a channel without peer slots")

    def send(self, req_id: int, shard_id: int, emb, last: bool = False) -> None:
        h = self.torch.tensor([req_id, shard_id, emb.shape[0], emb.shape[1], -1, 0, 0, 0], dtype=self.torch.int64)
        self.dist.send(h, 0, group=self._g(self.ctrl, self.rank))
        w2 = self.dist.isend(emb.contiguous(), 0, group=self._g(self.data, self.rank))
        self.outgoing.append((w2, emb))
        if self.device.type == "cuda":
            self.outgoing = [o for o in self.outgoing if not o[0].is_completed()]

    def poll(self):
        """Receiver: list of (req_id, shard_id, tensor) that arrived since the last call."""
        import queue
        done = []
        while True:
            try:
                item = self.ready.get_nowait()
            except queue.Empty:
                return done
            if item is None:
                self.ended += 1
            else:
                done.append(item)

    def close(self) -> None:
        if self.rank != 0:
            for w, _ in self.outgoing:
                w.wait()
            self.dist.send(self.torch.tensor([-1, -1, 0, 0, -1, 0, 0, 0], dtype=self.torch.int64), 0,
                           group=self._g(self.ctrl, self.rank))
        else:
            for th in self.threads:
                th.join(timeout=60)

    def finished_sources(self) -> int:
        return self.ended

    @staticmethod
    def _g(group, src):
        return group.get(src) if isinstance(group, dict) else group


class PeerShardChannel(ShardChannel):
    """ShardChannel whose payload bypasses NCCL (K9 + K10 fused, CUDA only).

    Rank 0 (the LLM-backend rank) owns ``n_slots`` receive slots per source rank in symmetric
    memory (torch.distributed._symmetric_memory: the same allocation mapped into every rank over
    NVLink).  A source's encoder packs its batch output straight into its next slot on rank 0
    (``alloc`` -> a peer view; K9 stages whole rows in shared memory and moves them with bulk
    copies, mmk_pack_mllama_peer), and once the batch has completed only the int64 header travels
    (gloo), naming slot and rows.  Rank 0 consumes the rows in place and releases the slot with a
    stream-ordered signal; the source's stream waits on that signal before packing into the slot
    again.  Batches larger than a slot fall back to the NCCL payload of the base class.  A tensor
    that ``poll`` returns for a slot aliases it: valid until the source has packed ``n_slots``
    more batches (consume it in ``on_receive`` / ``on_arrival``, which run before the release)."""

    def __init__(self, rank: int, world: int, device, dtype, slot_rows: int, width: int, n_slots: int = 2,
                 ctrl_group=None, data_group=None, on_arrival=None, on_receive=None, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        if torch.device(device).type != "cuda":
            raise RuntimeError("PeerShardChannel needs CUDA devices (NVLink peer memory)")
        self.slot_rows, self.width, self.n_slots = int(slot_rows), int(width), int(n_slots)
        self.slot_elems = self.slot_rows * self.width
        self.sym = symm.empty(world * self.n_slots * self.slot_elems, dtype=dtype, device=device)
        self.hdl = symm.rendezvous(self.sym, group if group is not None else dist.group.WORLD)
        self.uses = 0            # source: batches packed into peer slots so far
        self.open = {}           # source: slot -> (first byte address, bytes) of batches not yet sent
        super().__init__(rank, world, device, dtype, ctrl_group, data_group, on_arrival, on_receive)

    def _offset(self, src: int, slot: int) -> int:
        return (src * self.n_slots + slot) * self.slot_elems

    def alloc(self, rows: int, width: int):
        """Source rank: destination for a batch output of ``rows`` x ``width`` (a view of rank 0's
        memory), or None when it does not fit a slot (the caller packs locally; ``send`` then ships
        the payload over NCCL)."""
        if width != self.width or rows > self.slot_rows:
            return None
        slot = self.uses % self.n_slots
        if self.uses >= self.n_slots:  # stream-ordered: rank 0 released this slot's previous batch
            self.hdl.wait_signal(0, slot, 600000)
        self.uses += 1
        view = self.hdl.get_buffer(0, (rows, width), self.dtype, self._offset(self.rank, slot))
        self.open[slot] = (view.data_ptr(), rows * width * view.element_size())
        return view

    def send(self, req_id: int, shard_id: int, emb, last: bool = False) -> None:
        p = emb.data_ptr()
        slot = next((k for k, (base, n) in self.open.items() if base <= p < base + n), None)
        if slot is None:
            return super().send(req_id, shard_id, emb, last)
        row0 = (p - self.open[slot][0]) // (self.width * emb.element_size())
        h = self.torch.tensor([req_id, shard_id, emb.shape[0], emb.shape[1], slot, row0, int(last), 0],
                              dtype=self.torch.int64)
        self.dist.send(h, 0, group=self._g(self.ctrl, self.rank))
        if last:
            del self.open[slot]

    def _peer_arrival(self, src, rid, sid, rows, width, slot, row0, last):
        base = self._offset(src, slot) + row0 * width
        buf = self.sym[base:base + rows * width].view(rows, width)
        if self.on_receive is not None:
            self.on_receive(rid, sid, buf)
        extra = self.on_arrival(buf) if self.on_arrival is not None else None
        if last:  # every row of the slot handed on: release it, stream-ordered after the work above
            self.hdl.put_signal(src, slot)
        self.ready.put((rid, sid, buf if extra is None else extra))


@dataclass
class ReplayResult:
    latencies_ms: dict          # request id -> image-path latency (arrival -> all shards on rank 0)
    makespan_ms: float
    images: int
    batches: int

    def summary(self) -> dict:
        lat = list(self.latencies_ms.values())
        return {"requests": len(lat), "images": self.images, "batches": self.batches,
                "makespan_ms": round(self.makespan_ms, 3),
                "images_per_s": round(self.images / (self.makespan_ms / 1000.0), 3) if self.makespan_ms else None,
                "p50_ms": round(quantile(lat, 0.5), 3) if lat else None,
                "p90_ms": round(quantile(lat, 0.9), 3) if lat else None,
                "p99_ms": round(quantile(lat, 0.99), 3) if lat else None,
                "mean_ms": round(sum(lat) / len(lat), 3) if lat else None}


class ImagePathService:
    """One image instance per process (rank); rank 0 is also the LLM-backend (join) rank."""

    def __init__(self, spec: ModelSpec, executor=None, rank: int = 0, world: int = 1,
                 policies: pol.PolicySet | None = None, max_batch: dict | None = None, cost_ms=None,
                 ttft_slo_ms: float = 1e9, connector=None):
        self.spec, self.executor, self.rank, self.world = spec, executor, rank, world
        if executor is not None:
            # no graph capture under the service: receiver threads launch work concurrently (a
            # capture would see their launches) and trace batches rarely repeat a shape
            executor.graphs = False
        self.policies = policies or pol.PolicySet()
        self.max_batch = max_batch or {StageKind.ENCODE.value: 8}
        self.cost_ms = cost_ms or (lambda tiles: 10.0 * tiles)
        self.ttft_slo_ms = ttft_slo_ms
        self.connector = connector  # optional LLM-side projector applied on rank 0 as shards land
        self.projected = {}         # (request id, shard id) -> projected shape (outputs go to prefill, not kept)

    def plan(self, requests):
        """Per-rank WorkItems (one ENCODE item per routed shard) + shard counts per request."""
        routes = route_requests(requests, self.world, self.cost_ms, self.policies)
        by_id = {r.id: r for r in requests}
        items, shards_of = [], {}
        seq = 0
        for rid in sorted(routes, key=lambda i: (by_id[i].arrival_ms, i)):
            r = by_id[rid]
            shards_of[rid] = len(routes[rid])
            for sid, (inst, idx) in enumerate(routes[rid]):
                if inst != self.rank:
                    continue
                tiles = sum(r.images[i].tiles for i in idx)
                items.append(WorkItem(seq=seq, request_id=rid, stage=StageKind.ENCODE,
                                      size_tokens=sum(r.images[i].image_tokens for i in idx), tiles=tiles,
                                      enqueue_ms=r.arrival_ms, ttft_slo_ms=self.ttft_slo_ms,
                                      image_tokens=sum(r.images[i].image_tokens for i in idx),
                                      shard_images=tuple(idx), shard_id=sid))
                seq += 1
        return items, shards_of

    def replay(self, requests: list[Request], speed: float = 1.0, channel: ShardChannel | None = None,
               barrier=None) -> ReplayResult:
        """Replay ``requests`` in real time (trace ms / speed).  Needs a GPU executor."""
        import torch
        items, shards_of = self.plan(requests)
        by_id = {r.id: r for r in requests}
        images = {}
        for it in items:
            r = by_id[it.request_id]
            images.setdefault(it.request_id, {})
            for i in it.shard_images:
                im = r.images[i]
                images[it.request_id][i] = synthetic_image(r.id, i, im.width_px, im.height_px)
        # executor.run wants the request's image list; missing (other-rank) entries are never touched
        img_lists = {rid: [d.get(i) for i in range(len(by_id[rid].images))] for rid, d in images.items()}
        pending = sorted(items, key=lambda it: (it.enqueue_ms, it.seq))
        queue: list[WorkItem] = []
        arrived_at_0 = {}   # (rid, sid) -> ms on the replay clock
        inflight = None
        n_batches = 0
        if barrier is not None:
            barrier()
        t0 = time.perf_counter()
        clock = lambda: (time.perf_counter() - t0) * 1000.0 * speed  # noqa: E731
        nxt = 0
        expected = sum(shards_of.values()) if self.rank == 0 else 0
        while True:
            now = clock()
            while nxt < len(pending) and pending[nxt].enqueue_ms <= now:
                queue.append(pending[nxt])
                nxt += 1
            progressed = False
            if inflight is not None and inflight[1].query():
                batch, _, out = inflight
                t_done = clock()
                for k, it in enumerate(batch):
                    a, b = out.item_spans[it.seq]
                    rows0 = sum(out.image_tokens[:a])
                    rows1 = rows0 + sum(out.image_tokens[a:b])
                    if self.rank == 0:
                        arrived_at_0[(it.request_id, it.shard_id)] = t_done
                        if self.connector is not None:
                            y = self.connector(out.embeds[rows0:rows1])
                            self.projected[(it.request_id, it.shard_id)] = tuple(y.shape)
                    else:
                        channel.send(it.request_id, it.shard_id, out.embeds[rows0:rows1], last=k == len(batch) - 1)
                inflight = None
                progressed = True
            if inflight is None and queue:
                idx = form_batch(queue, now, self.policies.scheduler, self.policies.aging_slo_fraction,
                                 self.max_batch)
                if idx:
                    batch = [queue[i] for i in idx]
                    for i in sorted(idx, reverse=True):
                        queue.pop(i)
                    out_alloc = getattr(channel, "alloc", None) if self.rank != 0 else None
                    out = self.executor.run(batch, img_lists, out_alloc=out_alloc)
                    ev = torch.cuda.Event()
                    ev.record()
                    inflight = (batch, ev, out)
                    n_batches += 1
                    progressed = True
            if self.rank == 0 and channel is not None:
                for rid, sid, item in channel.poll():
                    arrived_at_0[(rid, sid)] = clock()
                    if self.connector is not None:
                        self.projected[(rid, sid)] = tuple(item.shape)
                    progressed = True
            mine_done = nxt == len(pending) and not queue and inflight is None
            if self.rank == 0:
                if mine_done and len(arrived_at_0) >= expected and (
                        channel is None or channel.finished_sources() == self.world - 1):
                    break
            elif mine_done:
                break
            if not progressed:
                time.sleep(0.0002)
        if channel is not None:
            channel.close()
        makespan = clock()
        lat = {}
        if self.rank == 0:
            for rid, n in shards_of.items():
                done = max(arrived_at_0[(rid, s)] for s in range(n))
                lat[rid] = done - by_id[rid].arrival_ms
        n_img = sum(len(by_id[rid].images) for rid in shards_of)
        return ReplayResult(latencies_ms=lat, makespan_ms=makespan, images=n_img, batches=n_batches)
