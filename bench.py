#!/usr/bin/env python
"""Image-path benchmark (preprocess + encode + pack) on 1..N B200s — the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mmk|reference] [--model M] [--batch B]

One step = one pass of the image path (K0 tile plan -> K1 preprocess -> encoder K2-K8 -> K9 pack)
over one batch of B synthetic images per GPU.  Default workload = BASELINE.json configs[1]:
Llama-3.2-11B-Vision encoder (560 px tiles, <= 4 tiles), image sizes drawn by the reference's
own workload generator (seed 0), random-init weights, bf16 compute / fp32 accumulate.

Prints ONE JSON line on rank 0.  ``value`` is whole-job images/s with the uint8 images already
resident in HBM; ``e2e`` is the same metric through the public API
(ImagePathExecutor.encode_images) from pinned host memory, with H2D of the images and a D2H of
the token offsets + a checksum of the packed embeddings inside the timed region.  For N > 1 each
rank encodes its own shard (weak scaling) and hands its packed embeddings to rank 0 (the
LLM-backend GPU) with NCCL point-to-point sends inside the timed region (BASELINE configs[3]).

Multi-GPU (``--gpus N`` under torchrun): the images are partitioned over the ranks by the path's
own data-parallel partition (dp.partition_images with per-image encoder FLOPs, the cost-weighted
form of the reference's split_by_tiles, policies.py:91-101) and every rank's packed rows are
handed to rank 0 inside the timed region.  ``--scaling weak`` (default): N x B images per step,
per-GPU work fixed; ``--scaling strong``: a fixed global batch (``--global-batch``) split N ways.

``--impl reference`` times the CPU implementation of the path (the oracle port in oracle/: the C
preprocess + torch fp32 encoder, all host threads) on the SAME workload: each step is one image
(one image per tile count present in the batch, in turn), and images/s is the batch's time
estimated from the per-tile-count means weighted by the batch's tile histogram.  It imports no
product CUDA code (libmmk is never mapped).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "llama3.2-11b": dict(config="Llama-3.2-11B-Vision image encoder, 560px tiles (<=4), bf16",
                         batch=32, generator=dict()),
    "llava-clip-l14-336": dict(config="LLaVA-style CLIP ViT-L/14-336, layer -2, CLS dropped, ragged packing",
                               batch=256, generator=dict()),
    "vit-b16-224": dict(config="reference default: 224x224 single tile -> ViT-B/16", batch=8, fixed=(224, 224)),
    "llava-ov-7b": dict(config="LLaVA-OneVision SigLIP-400M, 384px tiles (<=10) + thumbnail, bf16",
                        batch=32, generator=dict()),
    "internvl-26b": dict(config="InternVL-26B InternViT-6B, 448px tiles (<=5) + thumbnail, pixel shuffle, bf16",
                         batch=32, generator=dict()),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mmk", choices=["mmk", "reference"])
    ap.add_argument("--model", default="llama3.2-11b", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="images per GPU per step (0 = workload default)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: images per step over all GPUs (0 = 4 x the workload batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def image_dims(spec, n_images: int, seed: int = 0, fixed=None):
    """Image sizes from the reference generator (workload.py:247-252), image requests only."""
    if fixed is not None:
        return [tuple(fixed)] * n_images
    from paper_2502_00937_b200 import workload
    cfg = workload.GeneratorConfig(model=spec, base_rate=50.0, image_request_fraction=1.0, seed=seed)
    dims = []
    horizon = 10_000.0
    while len(dims) < n_images:
        dims = workload.image_dims_of(workload.generate(cfg, horizon))
        horizon *= 2
    return dims[:n_images]


def workload_dims(spec, wl, B, G, scaling):
    """Image sizes of one step over all GPUs.  Weak scaling: the N=1 batch's sizes repeated per GPU
    (new pixels for every copy), so the cost-balanced partition hands every rank the same work as
    the one-GPU step; strong scaling: the first G generator images."""
    if scaling == "weak":
        base = image_dims(spec, B, fixed=wl.get("fixed"))
        return [base[i % B] for i in range(G)]
    return image_dims(spec, G, fixed=wl.get("fixed"))


def make_images(dims, seed, first_index: int = 0):
    """Random uint8 pixels; image i of the workload is seeded by (seed, first_index + i), so an
    image has the same pixels whichever rank encodes it."""
    return [np.random.default_rng((seed, first_index + i)).integers(0, 256, (h, w, 3), dtype=np.uint8)
            for i, (w, h) in enumerate(dims)]


def images_at(dims, seed, indices):
    return [np.random.default_rng((seed, i)).integers(0, 256, (dims[i][1], dims[i][0], 3), dtype=np.uint8)
            for i in indices]


def encoder_flops(spec, tiles_list):
    """Algorithmic FLOPs of the encoder per image:
    F = L*S*(8d^2 + 4*d*ff) + 4*L*S^2*d + n_patch*2*(3p^2)*d, S = attention length of the image."""
    enc = spec.encoder
    P = (spec.tile_edge_px // enc.patch_px) ** 2
    if enc.family == "clip":
        L = enc.layers if enc.out_layer == -1 else enc.layers + 1 + enc.out_layer
    else:
        L = enc.layers + enc.global_layers
    d, ff = enc.hidden, enc.ffn
    tot = 0.0
    for t in tiles_list:
        S = t * spec.seq_per_tile
        # attention span: the whole image (Mllama), one tile (CLIP-family ViTs)
        attn = S * S if enc.family == "mllama" else t * spec.seq_per_tile ** 2
        tot += L * S * (8 * d * d + 4 * d * ff) + 4 * L * attn * d + t * P * 2 * (3 * enc.patch_px ** 2) * d
    return tot


def attention_exp_roofline(a, spec, clocks):
    """The attention's other bound: one exponential per score, 7 of every 8 on MUFU.EX2 (16 per
    clock per SM on B200: 8 cycles per warp instruction per sub-partition, scripts/micro/pipes.cu),
    1 of 8 on an FMA-pipe polynomial (speculative tiles).  MUFU ops/s achieved vs 16 x SMs x the
    median SM clock sampled during the timed region."""
    import torch
    if not a.get("ms") or not clocks.get("sm_mhz"):
        return None
    scores = a["work"] / (4.0 * spec.encoder.head_dim)  # work = 4 S^2 H hd with the model's head_dim
    mufu = scores * 7.0 / 8.0 / (a["ms"] / 1e3)
    peak = 16.0 * torch.cuda.get_device_properties(0).multi_processor_count * clocks["sm_mhz"] * 1e6
    return {"bound": "mufu", "achieved": round(mufu / 1e12, 3), "peak": round(peak / 1e12, 3), "unit": "Tops/s",
            "frac": round(mufu / peak, 4),
            "note": "exponentials of the attention (one per score, 7/8 on MUFU.EX2) per second vs the MUFU rate "
                    "at the sampled median SM clock"}


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def result(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops_sustained", 1398.9), d.get("bf16_tflops", 1646.7), d.get("hbm_gbs", 6548.2), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


def committed_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_reference_time(spec, imgs, weights, threads: int):
    """Seconds of the CPU path (oracle port: C preprocess + torch fp32 encoder) on these images."""
    import torch
    from oracle import encoders as oenc
    from oracle import preprocess as oprep
    from oracle import tiling as otiling
    from paper_2502_00937_b200.weights import k_pad_of
    torch.set_num_threads(threads)
    enc = spec.encoder
    dims = [(im.shape[1], im.shape[0]) for im in imgs]
    scale, shift = oprep.norm_constants(enc.mean, enc.std)
    t0 = time.perf_counter()
    plan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], spec.tile_edge_px, spec.tokens_per_tile,
                             spec.max_tiles_per_image, spec.thumbnail_tile, enc.resize_mode)
    patches = oprep.bf16_bits_to_f32(oprep.preprocess(imgs, plan, spec.tile_edge_px, enc.patch_px, k_pad_of(spec),
                                                      enc.resize_mode, spec.thumbnail_tile, scale, shift))
    out = oenc.encode(torch.from_numpy(patches), plan, weights, spec)
    _ = float(out.float().sum())
    return time.perf_counter() - t0


class MixSampler:
    """Same-config CPU sampling: one sample = one image of a tile count present in the batch (a
    group of up to 8 images when the batch has a single tile count); the batch's CPU time is
    estimated as sum over tile counts of (images with that count) x (mean seconds per image of
    that count), tile counts never sampled scaled from the sampled ones by encoder FLOPs."""

    def __init__(self, spec, dims, seed):
        from paper_2502_00937_b200 import core
        self.spec, self.dims, self.seed = spec, dims, seed
        self.tiles = [core.tile_count(w, h, spec) for w, h in dims]
        self.hist = {t: self.tiles.count(t) for t in sorted(set(self.tiles))}
        self.group = min(8, len(dims)) if len(self.hist) == 1 else 1
        self.order = sorted(self.hist, key=lambda t: -self.hist[t])  # most frequent tile count first
        self.by_count = {t: [i for i, x in enumerate(self.tiles) if x == t] for t in self.hist}
        self.times: dict = {t: [] for t in self.hist}
        self.k = 0

    def next_sample(self):
        t = self.order[self.k % len(self.order)]
        pool = self.by_count[t]
        start = (self.k // len(self.order)) * self.group
        idx = [pool[(start + j) % len(pool)] for j in range(self.group)]
        self.k += 1
        return t, images_at(self.dims, self.seed, idx)

    def record(self, t, seconds):
        self.times[t].append(seconds / self.group)

    def batch_seconds(self):
        per = {t: sum(v) / len(v) for t, v in self.times.items() if v}
        flops = {t: encoder_flops(self.spec, [t]) for t in self.hist}
        ref_t = max(per, key=lambda t: len(self.times[t]))
        est = {t: per.get(t, per[ref_t] * flops[t] / flops[ref_t]) for t in self.hist}
        return sum(self.hist[t] * est[t] for t in self.hist), est

    def describe(self, est):
        return {"tile_histogram": {str(t): c for t, c in self.hist.items()},
                "seconds_per_image": {str(t): round(v, 3) for t, v in est.items()},
                "samples": {str(t): len(v) * self.group for t, v in self.times.items()},
                "same_config": True}


def cpu_baseline_line(spec, dims, weights, seed, threads, budget_s: float = 60.0, per_count: int = 2):
    """``per_count`` samples (different images) per tile count of the batch (at least
    two), one pass over the counts at a time, most frequent first, until ~``budget_s`` of CPU work
    (Mllama: ~43 s; InternViT-6B, ~10 s per tile, stops earlier); the batch time is weighted by the
    batch mix, tile counts left unsampled scaled by encoder FLOPs."""
    ms = MixSampler(spec, dims, seed)
    spent = 0.0
    for _ in range(per_count * len(ms.hist)):
        if spent > budget_s:
            break
        t, imgs = ms.next_sample()
        dt = cpu_reference_time(spec, imgs, weights, threads)
        ms.record(t, dt)
        spent += dt
    total, est = ms.batch_seconds()
    return {"value": round(len(dims) / total, 4), "unit": "images/s", "cores": threads, "kind": "port",
            "sample": f"{ms.group} image(s) per sample, up to {per_count} samples per tile count of the {len(dims)}-image "
                      f"batch (see samples), CPU time of the batch "
                      f"estimated from the per-tile-count seconds weighted by its tile histogram (oracle C "
                      f"preprocess + torch fp32 encoder, {threads} threads)",
            **ms.describe(est)}


def run_reference(args, spec, wl, rank, world, out=None):
    """--impl reference: CPU implementation of the path on this box's host cores (rank 0 only),
    on the GPU arm's workload (same image sizes and pixels), with no product CUDA code loaded."""
    if rank != 0:
        return
    from paper_2502_00937_b200.weights import init_weights
    threads = len(os.sched_getaffinity(0))
    weights = init_weights(spec, 0)
    B = args.batch or wl["batch"]
    G = B * world if args.scaling == "weak" else (args.global_batch or 4 * B)
    dims = workload_dims(spec, wl, B, G, args.scaling)
    ms = MixSampler(spec, dims, 1000)
    step_s = []
    for s_i in range(args.warmup + args.steps):
        t, imgs = ms.next_sample()
        dt = cpu_reference_time(spec, imgs, weights, threads)
        if s_i >= args.warmup:
            ms.record(t, dt)
            step_s.append(dt)
    total, est = ms.batch_seconds()
    val = G / total
    maps = open("/proc/self/maps").read() if os.path.exists("/proc/self/maps") else ""
    native = sorted({ln.split()[-1] for ln in maps.splitlines() if ln.endswith(".so") and ROOT in ln})
    assert not any("libmmk" in x for x in native), native  # the reference arm never maps product CUDA code
    line = {
        "impl": "reference", "metric": "images/sec (preprocess+encode)", "value": round(val, 4), "unit": "images/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * sum(step_s) / max(1, len(step_s)), 3),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl["config"], "model": spec.name, "images_per_step_of_gpu_arm": G,
                   "image_dims": "reference generator seed 0 (the GPU arm's batch)", "step": "one CPU sample"},
        "cpu_baseline": {"value": round(val, 4), "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": f"{ms.group} image(s) per step, cycling over the tile counts of the GPU arm's "
                                   f"{G}-image batch; batch time = per-tile-count mean seconds x its tile histogram "
                                   f"(oracle C preprocess + torch fp32 encoder on {threads} threads)",
                         **ms.describe(est)},
        "native_so_loaded": native,
        "e2e": {"value": round(val, 4), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=out or sys.stdout, flush=True)


# ----------------------------------------------------------------------------- GPU path
def _reserve_stdout_for_result():
    """The driver parses exactly one JSON line from stdout: send everything else (NCCL's banner,
    library prints) to stderr and keep a private handle on the real stdout for the result."""
    sys.stdout.flush()
    fd = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(fd, "w", buffering=1)


def main():
    args = parse()
    result_out = _reserve_stdout_for_result()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2502_00937_b200 import core
    spec = core.get_model_spec(args.model)
    wl = WORKLOADS[args.model]
    if args.impl == "reference":
        return run_reference(args, spec, wl, rank, world, out=result_out)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2502_00937_b200 import ops
    from paper_2502_00937_b200.dp import Handoff, partition_images
    from paper_2502_00937_b200.executor import ImagePathExecutor, stage_images

    B = args.batch or wl["batch"]
    # the step's images: weak scaling N x B (per-GPU work fixed), strong scaling a fixed global
    # batch; partitioned over the ranks by the path's own DP partition weighted by encoder FLOPs
    G = B * world if args.scaling == "weak" else (args.global_batch or 4 * B)
    all_dims = workload_dims(spec, wl, B, G, args.scaling)
    all_tiles = [core.tile_count(w, h, spec) for w, h in all_dims]
    shards = partition_images(all_tiles, world, costs=[encoder_flops(spec, [t]) for t in all_tiles])
    mine = shards[rank]
    dims = [all_dims[i] for i in mine]
    imgs = images_at(all_dims, 1000, mine)
    # narrow encoders (ViT-B) fold their LayerNorms only when configured for large batches (the
    # executor's choice is fixed, so embeddings stay batch-invariant): +7 % at 256 images, -2 % at 8
    fold = None if spec.encoder.hidden >= 1024 else B * spec.seq_per_tile >= 16384
    ex = ImagePathExecutor(spec, seed=0, fold_ln=fold)
    staged = stage_images(imgs)  # resident uint8 images in HBM (the `value` leg)
    tiles = [all_tiles[i] for i in mine]
    flops_per_step = encoder_flops(spec, tiles)
    flops_job = encoder_flops(spec, all_tiles)
    # the receiver computes every source's row count itself from the deterministic plan
    rank_rows = {r: sum(all_tiles[i] for i in shards[r]) * spec.tokens_per_tile for r in range(world)}
    # handoff of every rank's packed rows to the LLM-backend rank 0: K9+K10 fused (each rank's
    # pack writes its rows straight into its region of rank 0's symmetric-memory prefill buffer
    # over NVLink); NCCL point-to-point (dp.Handoff) if symmetric memory is unavailable
    handoff, out_alloc, handoff_kind = None, None, None
    if world > 1:
        try:
            import torch.distributed._symmetric_memory as symm
            enc = spec.encoder
            width = enc.out_width
            first = [sum(rank_rows[q] for q in range(r)) * width for r in range(world)]
            prefill = symm.empty(sum(rank_rows.values()) * width, dtype=torch.bfloat16, device="cuda")
            hdl = symm.rendezvous(prefill, dist.group.WORLD)
            my_slot = hdl.get_buffer(0, (rank_rows[rank], width), torch.bfloat16, first[rank])

            def out_alloc(rows, w, _slot=my_slot):
                assert (rows, w) == tuple(_slot.shape), (rows, w, tuple(_slot.shape))
                return _slot
            handoff_kind = "nvlink-pack-into-rank0"
        except Exception as exc:  # noqa: BLE001 — no peer memory: NCCL send/recv instead
            if rank == 0:
                print(f"symmetric memory unavailable ({str(exc)[:120]}); NCCL handoff", file=sys.stderr)
            handoff, handoff_kind = Handoff(rank, world), "p2p-handoff-to-rank0"
    stream = torch.cuda.current_stream()

    def step(batch):
        out = ex.encode(batch, out_alloc=out_alloc)
        if handoff is not None:
            handoff.send(out, sizes=rank_rows)
        return out

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the step as one CUDA graph (K0 -> K9, ~290 launches for Mllama): replayed in the timed region
    captured = ex.capture(staged, out_alloc=out_alloc)

    def step_graph():
        if handoff is not None:  # the replay rewrites the buffer earlier sends may still be reading
            handoff.release(captured.output.embeds)
        out = captured.replay()
        if handoff is not None:
            handoff.send(out, sizes=rank_rows)
        return out

    for _ in range(args.warmup):
        step_graph()
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            step_graph()
        if handoff is not None:
            handoff.flush()
        end.record(stream)
        barrier()
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = G * args.steps / (ms_max / 1000.0)

    # --------------------------------------------------------------- e2e through the public API
    # the step's inputs sit in pinned host memory (as a decoder writing page-locked buffers would
    # leave them); every step copies them to the device inside the timed region
    pinned_imgs = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in imgs]
    ck = torch.empty(1, device="cuda")
    for _ in range(2):  # a shape seen twice is captured by encode_images (outside the timed region)
        o = ex.encode_images(pinned_imgs, out_alloc=out_alloc)
        ops.checksum(o.embeds, out=ck)
    graphed = bool(ex._graph_cache) and out_alloc is None
    barrier()
    h2d = d2h = 0
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e_start.record(stream)
    for s_i in range(args.steps):
        o = ex.encode_images(pinned_imgs, out_alloc=out_alloc)
        # pixels; the eager path (a peer out_alloc) also copies the 16-byte per-image metadata
        h2d += sum(t_.numel() for t_ in pinned_imgs) + (0 if graphed else 16 * len(pinned_imgs))
        if handoff is not None:
            handoff.send(o, sizes=rank_rows)
        ops.checksum(o.embeds, out=ck)
        offs = o.tok_offsets.to("cpu", non_blocking=True)
        cks = ck.to("cpu", non_blocking=True)
        d2h += offs.numel() * 8 + 4
    if handoff is not None:
        handoff.flush()
    e_end.record(stream)
    barrier()
    e_ms = e_start.elapsed_time(e_end)
    t = torch.tensor([e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e_value = G * args.steps / (float(t.item()) / 1000.0)
    assert np.isfinite(float(cks.item()))

    # fixed-size workloads (the reference default, 224x224 single tiles): the path a server with a
    # fixed batch shape would take — the step captured once, then per step one H2D of the
    # page-locked batch into the captured input buffer and a replay (reported as e2e_graph)
    e2e_graph = None
    if wl.get("fixed"):
        host_batch = torch.cat([t_.reshape(-1) for t_ in pinned_imgs]).pin_memory()
        cap_e2e = ex.capture(stage_images(pinned_imgs), out_alloc=out_alloc)
        barrier()
        g_start, g_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g_start.record(stream)
        for _ in range(args.steps):
            if handoff is not None:
                handoff.release(cap_e2e.output.embeds)
            cap_e2e.batch.src.copy_(host_batch, non_blocking=True)
            o = cap_e2e.replay()
            if handoff is not None:
                handoff.send(o, sizes=rank_rows)
            ops.checksum(o.embeds, out=ck)
            cks = ck.to("cpu", non_blocking=True)
        if handoff is not None:
            handoff.flush()
        g_end.record(stream)
        barrier()
        t = torch.tensor([g_start.elapsed_time(g_end)], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_graph = {"value": round(G * args.steps / (float(t.item()) / 1000.0), 3), "unit": "images/s",
                     "h2d_bytes_per_step": int(host_batch.numel()), "d2h_bytes_per_step": 4,
                     "path": "ImagePathExecutor.capture(...).replay() after one H2D of the page-locked batch into "
                             "its input buffer + checksum D2H"}

    # --------------------------------------------------------------- e2e from JPEG bytes (GPU decode)
    e2e_jpeg = None
    try:
        from torchvision.io import encode_jpeg
        jpegs = [encode_jpeg(torch.from_numpy(np.ascontiguousarray(im.transpose(2, 0, 1))), quality=90) for im in imgs]
        o = ex.encode_jpegs(jpegs)
        barrier()
        j_start, j_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        jb = 0
        j_start.record(stream)
        for _ in range(args.steps):
            o = ex.encode_jpegs(jpegs)
            ops.checksum(o.embeds, out=ck)
            offs = o.tok_offsets.to("cpu", non_blocking=True)
            jb = sum(int(j.numel()) for j in jpegs)
        j_end.record(stream)
        barrier()
        t = torch.tensor([j_start.elapsed_time(j_end)], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_jpeg = {"value": round(G * args.steps / (float(t.item()) / 1000.0), 3), "unit": "images/s",
                    "h2d_bytes_per_step": jb, "path": "ImagePathExecutor.encode_jpegs (nvJPEG decode on the GPU)"}
    except Exception as exc:  # torchvision without CUDA JPEG support: report why
        if os.environ.get("BENCH_DEBUG"):
            import traceback
            traceback.print_exc()
        e2e_jpeg = {"unavailable": str(exc)[:200]}

    # per-kernel CUDA-event durations (after the e2e legs, so value and e2e are measured in the same
    # thermal state): the same K steps launched eagerly with an event pair
    # around every libmmk launch on the launching stream (roofline numerator / denominator)
    log = ops.LaunchLog(timing=True)
    ops.LOG = log
    i_start, i_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    i_start.record(stream)
    for _ in range(args.steps):
        step(staged)
    if handoff is not None:
        handoff.flush()
    i_end.record(stream)
    barrier()
    ops.LOG = None
    ms_instr = i_start.elapsed_time(i_end)
    kernels = log.summary()
    launches = log.count

    if rank == 0:
        sus, burst, hbm, src = measured_peaks()
        g = kernels.get("gemm", {"ms": 0, "work": 0, "launches": 0})
        a = kernels.get("attention", {"ms": 0, "work": 0, "launches": 0})
        traffic = committed_traffic().get(spec.name, {})
        step_ms = ms_max / args.steps
        # dominant kernel = the single kernel kind with the largest share of the (instrumented)
        # step: attention, or one GEMM form (QKV bf16 / FC1+act / residual) — not the GEMM family
        subs = {k: v for k, v in kernels.items() if k.startswith("gemm.") and v["ms"]}
        top_sub = max(subs, key=lambda k: subs[k]["ms"]) if subs else "gemm"
        dominant = "attention" if a["ms"] >= subs.get(top_sub, g)["ms"] else top_sub
        names = {"gemm": "mmk gemm_bf16_tcgen05(_2sm): persistent TMA + tcgen05 (CTA pairs), fused epilogues",
                 "attention": "mmk attn_fwd_tc(_persistent): varlen flash attention, S/O/P in TMEM, tcgen05 + TMA, "
                              "speculative row max"}

        def roof_entry(kind):
            k = a if kind == "attention" else kernels.get(kind, g)
            tf = k["work"] / (k["ms"] / 1e3) / 1e12 if k["ms"] else 0.0
            name = names["attention"] if kind == "attention" else names["gemm"] + ("" if kind == "gemm" else f" [{kind}]")
            return {"kernel": name, "bound": "tensor", "achieved": round(tf, 1), "peak": sus, "unit": "TFLOP/s",
                    "frac": round(tf / sus, 4) if sus else None, "peak_kind": f"{src} sustained bf16",
                    "traffic": traffic.get(kind, {}).get("bytes_per_launch"),
                    "traffic_note": traffic.get(kind, {}).get("note"),
                    "launches": k["launches"], "share_of_step": round(k["ms"] / ms_instr, 4) if ms_instr else None,
                    "timing": "per-launch CUDA events, eager repeat of the timed steps"}

        clocks = clk.result()
        enc_tf = flops_job / world / (step_ms / 1e3) / 1e12  # per GPU
        line = {
            "metric": "images/sec (preprocess+encode)", "value": round(value, 3), "unit": "images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference generator image sizes, random uint8 pixels, random-init weights)",
            "config": {"workload": wl["config"] + (f", data-parallel over {world} B200" if world > 1 else ""),
                       "model": spec.name, "images_per_step": G, "images_rank0": len(dims),
                       "graph": "one CUDA graph per step", "ln_fold": bool(ex.encoder.fold_ln),
                       "tiles_per_step": int(sum(all_tiles)), "tiles_rank0": int(sum(tiles)),
                       "tile_histogram": {str(t): all_tiles.count(t) for t in sorted(set(all_tiles))},
                       "tokens_per_step": int(sum(all_tiles)) * spec.tokens_per_tile,
                       "partition": "dp.partition_images(costs=encoder FLOPs per image) (cost-weighted "
                                    "split_by_tiles, reference policies.py:91-101)",
                       "l2": "inputs > L2 (activations of one step are several GB)",
                       "parallelism": f"dp{world}" + (f"+{handoff_kind}" if world > 1 else "")},
            "roofline": roof_entry(dominant),
            "roofline_other": {kind: roof_entry(kind) for kind in ["attention", "gemm", *sorted(subs)] if kind != dominant},
            "roofline_step": {"achieved": round(enc_tf, 1), "peak": sus, "unit": "TFLOP/s",
                              "frac": round(enc_tf / sus, 4),
                              "note": "algorithmic encoder FLOPs of the whole step / step time"},
            "roofline_attention_exp": attention_exp_roofline(a, spec, clocks),
            "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                            "achieved": round(v["work"] / (v["ms"] / 1e3) /
                                              (1e12 if (k in ("gemm", "attention") or k.startswith("gemm.")) else 1e9), 1)
                            if v["ms"] else None,
                            "unit": "TFLOP/s" if (k in ("gemm", "attention") or k.startswith("gemm.")) else "GB/s"}
                        for k, v in kernels.items()},
            "gpu_launches": launches,
            "e2e": {"value": round(e_value, 3), "unit": "images/s", "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": d2h // args.steps,
                    "path": ("ImagePathExecutor.encode_images(pinned host uint8 images): per-image H2D, then the "
                             "batch shape's captured graph replayed (eager launches with a peer out_alloc) + "
                             "token offsets and checksum D2H")},
            "e2e_graph": e2e_graph,
            "e2e_jpeg": e2e_jpeg,
            "clocks": clocks,
        }
        if not args.no_cpu_baseline and world == 1:
            w_cpu = {k: (v.cpu() if isinstance(v, torch.Tensor) else v) for k, v in ex.weights.items()}
            line["cpu_baseline"] = cpu_baseline_line(spec, all_dims, w_cpu, 1000, len(os.sched_getaffinity(0)))
        print(json.dumps(line), file=result_out, flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
