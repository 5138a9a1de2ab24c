"""Multi-process host logic of the DP path (world size 2, gloo on CPU): image partition and the
embedding handoff to the LLM-backend rank, with receiver-side sizing from the tile plan."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_00937_b200 import core
from paper_2502_00937_b200.dp import Handoff, partition_images


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = core.get_model_spec("llama3.2-11b")
    dims = [(560, 560), (1200, 700), (300, 2000), (1120, 1120), (800, 600), (64, 64)]
    tiles = [core.tile_count(w, h, spec) for w, h in dims]
    shards = partition_images(tiles, world)
    mine = shards[rank]
    rows = {r: sum(tiles[i] for i in shards[r]) * spec.tokens_per_tile for r in range(world)}
    width = 16
    # each rank's "packed embeddings": value = global image index, per token row
    emb = torch.cat([torch.full((tiles[i] * spec.tokens_per_tile, width), float(i)) for i in mine]) if mine \
        else torch.zeros(0, width)
    h = Handoff(rank, world, dst=0)
    for step in range(3):  # exercise the two-deep buffer ring
        h.send(emb + step, sizes=rows, width=width)
    h.flush()
    if rank == 0:
        got = {src: buf.clone() for src, buf in h.received.items()}
        ok = True
        for src, buf in got.items():
            expect = torch.cat([torch.full((tiles[i] * spec.tokens_per_tile, width), float(i)) for i in shards[src]]
                               + [torch.zeros(0, width)])
            ok &= torch.equal(buf, expect + 2)
        q.put((ok, [sorted(s) for s in shards]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_partition_and_handoff_gloo(world):
    """World 8 with 6 images: two ranks hold empty shards (zero-row sends and receives)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, shards = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert sorted(i for s in shards for i in s) == list(range(6))


def test_partition_images_shapes():
    assert partition_images([4, 1, 1, 2], 3) == [[0], [3], [1, 2]]
    assert partition_images([1], 4) == [[0], [], [], []]
    shards = partition_images([1, 2, 3, 4], 2, costs=[1.0, 5.0, 12.0, 20.0])
    assert sorted(i for s in shards for i in s) == [0, 1, 2, 3]


def _release_worker(rank, world, port, q):
    """A sender that reuses ONE output buffer (a replayed CUDA graph's) calls release() before
    rewriting it, so every step's rows arrive intact (write-after-read on replay)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, width = 64, 8
    h = Handoff(rank, world, dst=0, depth=3)
    buf = torch.zeros(rows, width)
    ok = True
    for step in range(5):
        h.release(buf)
        buf.fill_(float(step))  # the "replay" rewriting the captured output
        h.send(buf, sizes={1: rows}, width=width)
        if rank == 0:
            h.flush()
            ok &= torch.equal(h.received[1], torch.full((rows, width), float(step)))
        assert len(h.pending) <= 3
    h.flush()
    if rank == 0:
        q.put(ok)
    dist.barrier()
    dist.destroy_process_group()


def test_release_orders_buffer_reuse_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_release_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
