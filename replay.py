#!/usr/bin/env python
"""BASELINE configs[4]: bursty heavy-tailed multimodal trace (1-8 images/request) replayed in real
time through the modality-aware batcher on 1..N B200 (one image instance per GPU, rank 0 is
also the LLM-backend rank that joins the shards).

    python replay.py [--duration-s 20] [--rate 10] [--burst-mult 3] [--max-batch 8]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 replay.py ...

Prints one JSON line (rank 0): image-path latency percentiles (nearest-rank, reference
metrics.py:12-18), achieved images/s, batches, plus the trace description.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

IMAGES_PER_REQUEST = {1: 0.30, 2: 0.20, 3: 0.15, 4: 0.10, 5: 0.10, 6: 0.05, 7: 0.05, 8: 0.05}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3.2-11b")
    ap.add_argument("--duration-s", type=float, default=20.0)
    ap.add_argument("--rate", type=float, default=8.0, help="requests/s per GPU outside bursts")
    ap.add_argument("--burst-mult", type=float, default=3.0)
    ap.add_argument("--max-batch", type=int, default=8)
    ap.add_argument("--scheduler", default="slo_priority", choices=["fifo", "slo_priority"])
    ap.add_argument("--profile", default=None,
                    help="measured profile for the router's cost model (default profiles/measured_<model>.json; "
                         "measured on this GPU at start-up when absent)")
    ap.add_argument("--ms-per-tile", type=float, default=None,
                    help="override: a linear routing cost model instead of the measured profile")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--connector", action="store_true", help="apply the LLM-side projector on rank 0 as shards land")
    ap.add_argument("--handoff", default="peer", choices=["peer", "nccl"],
                    help="peer: encoders pack straight into rank 0's memory over NVLink (PeerShardChannel); "
                         "nccl: pack locally + NCCL send")
    ap.add_argument("--slot-images", type=int, default=16,
                    help="peer slot size in max-tile images (larger batches fall back to NCCL)")
    ap.add_argument("--verify", action="store_true",
                    help="rank 0 re-encodes every remote shard and compares it bit for bit with what arrived")
    ap.add_argument("--watchdog-s", type=float, default=0.0, help="dump all thread stacks after this many seconds")
    args = ap.parse_args()
    if args.watchdog_s > 0:
        import faulthandler
        faulthandler.dump_traceback_later(args.watchdog_s, exit=True)

    import torch
    import torch.distributed as dist
    from paper_2502_00937_b200 import core, policies, workload
    from paper_2502_00937_b200.executor import ImagePathExecutor
    from paper_2502_00937_b200.service import ImagePathService, PeerShardChannel, ShardChannel, route_requests

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    result_out = sys.stdout
    if world > 1:
        sys.stdout.flush()
        result_out = os.fdopen(os.dup(1), "w", buffering=1)  # NCCL banners -> stderr
        os.dup2(2, 1)
        # lazy NCCL communicator init: the per-source two-rank groups are created collectively
        # below and each connects on its first transfer
        dist.init_process_group("nccl")
    spec = core.get_model_spec(args.model)
    horizon = args.duration_s * 1000.0
    burst = workload.BurstEpisode(start_ms=0.4 * horizon, duration_ms=0.2 * horizon, rate_multiplier=args.burst_mult)
    cfg = workload.GeneratorConfig(model=spec, base_rate=args.rate * world, image_request_fraction=1.0,
                                   images_per_request=dict(IMAGES_PER_REQUEST), burst_episodes=(burst,),
                                   seed=args.seed)
    reqs = workload.generate(cfg, horizon)
    ex = ImagePathExecutor(spec, seed=0)
    # warm the executor (kernel attributes, allocator) outside the replay clock
    import numpy as np
    ex.encode_images([np.zeros((560, 560, 3), np.uint8)] * 2)
    torch.cuda.synchronize()
    pol = policies.PolicySet(router=policies.RouterKind.LEAST_PENDING,
                             scheduler=policies.SchedulerKind(args.scheduler), max_fanout=8, aging_slo_fraction=0.5)
    connector = None
    if args.connector and rank == 0:
        from paper_2502_00937_b200.connector import Projector
        connector = Projector(spec)
    # the router's cost model: the B200-measured encode latency (MeasuredProfile, the reference's
    # encode_latency seam, piecewise linear over batch tiles) — every rank loads / measures the
    # same profile so their deterministic routing agrees
    from paper_2502_00937_b200.profiles import MeasuredProfile, measure_profile
    if args.ms_per_tile is not None:
        cost_ms, cost_src = (lambda tiles: args.ms_per_tile * tiles), f"linear {args.ms_per_tile} ms/tile"
    else:
        path = args.profile or os.path.join(ROOT, "profiles", f"measured_{spec.name}.json")
        if os.path.exists(path):
            prof = MeasuredProfile.from_dict(json.loads(open(path).read()), spec)
            cost_src = f"measured profile {os.path.relpath(path, ROOT)}"
        else:
            prof = measure_profile(ex, batch_sizes=(1, 4, 16), iters=3, per_count_batch=4)
            if world > 1:  # one profile for every rank's router
                obj = [prof.to_dict()]
                dist.broadcast_object_list(obj, src=0)
                prof = MeasuredProfile.from_dict(obj[0], spec)
            cost_src = "measured at start-up"
        cost_ms = lambda tiles: prof.encode_latency(max(1, tiles), 1)  # noqa: E731
    svc = ImagePathService(spec, ex, rank=rank, world=world, policies=pol, max_batch={"encode": args.max_batch},
                           cost_ms=cost_ms, ttft_slo_ms=2000.0, connector=connector)
    chan = None
    digests = {}

    def digest(x):
        v = x.contiguous().view(torch.int16).reshape(-1).long()
        w = torch.arange(v.numel(), device=v.device) % 65521 + 1
        return torch.stack([v.sum(), (v * w).sum()])

    def on_receive(rid, sid, buf):  # receiver thread, before the slot is released
        digests[(rid, sid)] = (digest(buf), tuple(buf.shape))

    if world > 1:
        ctrl_g, data_g = ShardChannel.make_groups(world)
        # remote shards are projected by the receiver threads, on their own streams, as they land
        kw = dict(ctrl_group=ctrl_g, data_group=data_g, on_arrival=connector,
                  on_receive=on_receive if args.verify else None)
        dev = torch.device("cuda", local)
        if args.handoff == "peer":
            enc = spec.encoder
            P1 = spec.tokens_per_tile  # emitted rows per tile (InternVL: 256 of its 1025 encoder tokens)
            width = enc.out_width
            chan = PeerShardChannel(rank, world, dev, torch.bfloat16, slot_rows=args.slot_images * spec.max_tiles_per_image * P1,
                                    width=width, **kw)
        else:
            chan = ShardChannel(rank, world, dev, torch.bfloat16, **kw)
    res = svc.replay(reqs, channel=chan, barrier=(dist.barrier if world > 1 else None))
    if rank == 0:
        s = res.summary()
        n_img = sum(len(r.images) for r in reqs)
        line = {"metric": "image-path latency under a bursty trace", "n_gpus": world, **s,
                "trace": {"generator": "reference workload.generate", "seed": args.seed, "duration_s": args.duration_s,
                          "rate_req_s": args.rate * world, "burst": [burst.start_ms, burst.duration_ms, burst.rate_multiplier],
                          "images_per_request": IMAGES_PER_REQUEST, "requests": len(reqs), "images": n_img},
                "batcher": {"router": "least_pending", "scheduler": args.scheduler, "max_batch_encode": args.max_batch,
                            "router_cost_model": cost_src},
                "connector": (f"{spec.name} multi_modal_projector ({spec.encoder.out_width} -> 4096) on rank 0"
                              if args.connector else None),
                "handoff": (args.handoff if world > 1 else None),
                "handoff_shards": (dict(chan.counts) if chan is not None else None),
                "model": spec.name}
        if args.verify and world > 1:
            torch.cuda.synchronize()
            routes = route_requests(reqs, world, svc.cost_ms, svc.policies)
            by_id = {r.id: r for r in reqs}
            from paper_2502_00937_b200.service import synthetic_image
            bad = 0
            for (rid, sid), (dg, shape) in sorted(digests.items()):
                _, idx = routes[rid][sid]
                r = by_id[rid]
                imgs = [synthetic_image(rid, i, r.images[i].width_px, r.images[i].height_px) for i in idx]
                ref = ex.encode_images(imgs).embeds
                bad += int(tuple(ref.shape) != shape or not torch.equal(digest(ref), dg))
            line["verify"] = {"remote_shards": len(digests), "mismatches": bad}
        print(json.dumps(line), file=result_out, flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
