"""Replay-service host logic on CPU: deterministic least-pending routing (reference route_image
over a modelled instance state), per-rank WorkItem planning, and the streamed shard channel
over gloo with world size 2."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_00937_b200 import core, workload
from paper_2502_00937_b200.service import ImagePathService, ShardChannel, quantile, route_requests


def _reqs():
    spec = core.get_model_spec("llama3.2-11b")
    cfg = workload.GeneratorConfig(model=spec, base_rate=20.0, image_request_fraction=1.0,
                                   images_per_request={1: .4, 2: .3, 4: .2, 8: .1}, seed=3)
    return spec, workload.generate(cfg, 5000.0)


def test_quantile_matches_reference_rule():
    vals = [5, 1, 4, 2, 3]
    assert quantile(vals, 0.5) == 3 and quantile(vals, 0.99) == 5 and quantile(vals, 0.0) == 1
    assert quantile(list(range(1, 101)), 0.99) == 99


def test_routing_is_deterministic_and_complete():
    spec, reqs = _reqs()
    a = route_requests(reqs, 4, lambda t: 5.0 * t)
    b = route_requests(reqs, 4, lambda t: 5.0 * t)
    assert a == b
    for r in reqs:
        shards = a[r.id]
        assert sorted(i for _, idx in shards for i in idx) == list(range(len(r.images)))
        assert len(shards) == min(len(r.images), 4)
        assert len({inst for inst, _ in shards}) == len(shards)
    # per-rank plans partition all shards
    total = 0
    for rank in range(4):
        items, shards_of = ImagePathService(spec, rank=rank, world=4, cost_ms=lambda t: 5.0 * t).plan(reqs)
        total += len(items)
        assert all(it.shard_images for it in items)
    assert total == sum(len(v) for v in a.values())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _chan_worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    ch = ShardChannel(rank, 2, torch.device("cpu"), torch.float32)
    if rank == 1:
        for k in (3, 1, 2):  # out of order, variable sizes
            ch.send(100 + k, k, torch.full((k * 5, 4), float(k)))
        ch.close()
    else:
        got = {}
        while ch.finished_sources() < 1:
            for rid, sid, t in ch.poll():
                got[(rid, sid)] = t.clone()
        q.put(sorted((k, tuple(v.shape), float(v[0, 0])) for k, v in got.items()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_channel_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_chan_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [((101, 1), (5, 4), 1.0), ((102, 2), (10, 4), 2.0), ((103, 3), (15, 4), 3.0)]


class _SlotRecordingChannel(ShardChannel):
    """CPU stand-in for PeerShardChannel's header protocol: a header naming a slot carries no
    payload and is handed to ``_peer_arrival`` (the CUDA class maps it onto symmetric memory)."""

    def send_slot_header(self, rid, sid, rows, width, slot, row0, last):
        h = torch.tensor([rid, sid, rows, width, slot, row0, int(last), 0], dtype=torch.int64)
        self.dist.send(h, 0, group=self._g(self.ctrl, self.rank))

    def _peer_arrival(self, src, rid, sid, rows, width, slot, row0, last):
        self.ready.put((rid, sid, torch.tensor([src, rows, width, slot, row0, int(last)])))


def _slot_worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    ch = _SlotRecordingChannel(rank, 2, torch.device("cpu"), torch.float32)
    if rank == 1:
        ch.send_slot_header(7, 0, 1601, 7680, 1, 0, False)
        ch.send(8, 0, torch.full((3, 4), 2.0))            # payload path in between
        ch.send_slot_header(7, 1, 3202, 7680, 1, 1601, True)
        ch.close()
    else:
        got = {}
        while ch.finished_sources() < 1:
            for rid, sid, t in ch.poll():
                got[(rid, sid)] = t.tolist()
        q.put((sorted(got.items()), dict(ch.counts)))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_channel_slot_headers_gloo_world2():
    """The 8-int header: slot >= 0 means the rows are already in the receiver's memory."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_slot_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got, counts = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert counts == {"peer": 2, "nccl": 1}
    assert got == [((7, 0), [1, 1601, 7680, 1, 0, 0]), ((7, 1), [1, 3202, 7680, 1, 1601, 1]),
                   ((8, 0), [[2.0] * 4] * 3)]
