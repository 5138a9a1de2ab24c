"""ImagePathExecutor — the drop-in for the reference's modelled image stages.

In the reference simulator an image shard flows CPU lane -> GPU lane -> handoff:
``preprocess_latency`` (profiles.py:128-134, engine.py:639-657), then ``encode_latency``
(profiles.py:136-145, engine.py:682-716), then the shard join (engine.py:730-752) and the
transfer delay (engine.py:563-579).  Here the same batch objects (``WorkItem`` from
``form_batch``) are executed for real on one B200:

  stage (H2D of uint8 images) -> K0 tile plan -> K1 preprocess -> encoder (K2-K8) -> K9 pack

and the result is the packed prefill buffer [sum(image_tokens), D_out] bf16 plus int64
token offsets — exactly ``Request.total_image_tokens`` rows (core.py:110-112) per request.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .batcher import WorkItem
from .core import ModelSpec, SpecError, StageKind, tile_count
from .encoders import DeviceEncoder, init_weights
from .weights import DEVICE_INIT_PARAMS, param_count


@dataclass
class ImageBatch:
    """Raw images staged on the device: one flat uint8 HWC buffer + per-image metadata."""

    src: torch.Tensor          # uint8 [sum(h*w*3)]
    src_off: torch.Tensor      # int64 [n] byte offsets
    w: torch.Tensor            # int32 [n]
    h: torch.Tensor            # int32 [n]
    dims: list                 # host [(w, h)]
    h2d_bytes: int = 0
    chw: bool = False          # pixel layout of src: HWC (host decoders) or CHW planes (GPU JPEG decode)
    ready: "torch.cuda.Event | None" = None  # set when staged on a side stream: encode() waits on it
    parts: tuple = ()          # separately allocated images src_off points into (GPU JPEG decode)

    @property
    def src_bytes(self) -> int:
        return int(sum(w * h * 3 for w, h in self.dims))

    @property
    def n(self) -> int:
        return len(self.dims)


@dataclass
class PackedBatch:
    embeds: torch.Tensor                 # bf16 [sum tokens, D_out]  (LLM-prefill layout)
    tok_offsets: torch.Tensor            # int64 [n+1] device (from K0)
    tiles: list[int]                     # host, per image
    image_tokens: list[int]              # host, per image
    item_spans: dict = field(default_factory=dict)  # WorkItem.seq -> (first image, end image)

    @property
    def total_tokens(self) -> int:
        return int(sum(self.image_tokens))


def _as_hwc_u8(img) -> np.ndarray | torch.Tensor:
    if isinstance(img, torch.Tensor):
        if img.dtype != torch.uint8 or img.dim() != 3 or img.shape[2] != 3:
            raise SpecError("images must be uint8 HWC tensors with 3 channels")
        return img
    a = np.asarray(img)
    if a.dtype != np.uint8 or a.ndim != 3 or a.shape[2] != 3:
        raise SpecError("images must be uint8 HWC arrays with 3 channels")
    return a


def stage_images(images, device="cuda", pinned: bool = True, stream=None) -> ImageBatch:
    """Concatenate uint8 HWC images (host arrays or tensors) into one device buffer.

    stream: a side CUDA stream for the host-to-device copy, so staging the next batch overlaps
    the encode of the current one; ``ImagePathExecutor.encode`` waits on the copy's event."""
    imgs = [_as_hwc_u8(i) for i in images]
    dims = [(int(i.shape[1]), int(i.shape[0])) for i in imgs]
    for w, h in dims:
        if w < 1 or h < 1:
            raise SpecError("image dimensions must be >= 1 pixel")
    sizes = [w * h * 3 for w, h in dims]
    offs = np.zeros(len(imgs), np.int64)
    if imgs:
        offs[1:] = np.cumsum(sizes)[:-1]
    total = int(sum(sizes))
    dev = torch.device(device)
    meta = np.concatenate([offs.view(np.int32), np.array([d[0] for d in dims], np.int32),
                           np.array([d[1] for d in dims], np.int32)]) if imgs else np.zeros(0, np.int32)
    # images already in pinned host tensors (a decoder writing straight into page-locked memory)
    # are copied to the device one by one, without a host-side concatenation
    direct = bool(imgs) and all(isinstance(i, torch.Tensor) and i.device.type == "cpu" and i.is_pinned()
                                and i.is_contiguous() for i in imgs)
    host = None
    if not direct:
        host = torch.empty(total, dtype=torch.uint8, pin_memory=pinned)
        hv = host.numpy()
        for i, im in enumerate(imgs):
            a = im.cpu().numpy() if isinstance(im, torch.Tensor) else im
            hv[offs[i]:offs[i] + sizes[i]] = a.reshape(-1)
    hmeta = torch.from_numpy(meta)
    if pinned:
        hmeta = hmeta.pin_memory()

    def copy_in():
        if direct:
            dst = torch.empty(total, dtype=torch.uint8, device=dev)
            for i, im in enumerate(imgs):
                dst[offs[i]:offs[i] + sizes[i]].copy_(im.view(-1), non_blocking=True)
            return dst, hmeta.to(dev, non_blocking=True)
        return host.to(dev, non_blocking=True), hmeta.to(dev, non_blocking=True)

    ready = None
    if stream is not None:
        with torch.cuda.stream(stream):
            src, dmeta = copy_in()
            ready = torch.cuda.Event()
            ready.record(stream)
    else:
        src, dmeta = copy_in()
    n = len(imgs)
    src_off = dmeta[:2 * n].view(torch.int64)
    return ImageBatch(src=src, src_off=src_off, w=dmeta[2 * n:3 * n], h=dmeta[3 * n:4 * n], dims=dims,
                      h2d_bytes=total + meta.nbytes, ready=ready)


@dataclass
class CapturedEncode:
    graph: "torch.cuda.CUDAGraph"
    batch: ImageBatch
    output: PackedBatch

    def replay(self) -> PackedBatch:
        self.graph.replay()
        return self.output


class _GraphEntry:
    """One cached batch shape: the staged input buffer, the captured K0..K9 graph and its output.
    ``run`` copies new pixels in and replays; the returned tensors are fresh copies, so a result
    never changes under its holder when the shape is encoded again.  Pinned-tensor inputs go
    host-to-device on a copy stream into one of two landing buffers, so a call's H2D overlaps the
    previous call's replay; the compute stream then moves them into the graph's input buffer with
    one device copy.  Host arrays go through a page-locked staging copy."""

    def __init__(self, ex: "ImagePathExecutor", imgs: list):
        self.sizes = [int(im.shape[0]) * int(im.shape[1]) * 3 for im in imgs]
        self.offs = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.host = None       # page-locked staging copy for host arrays (lazily)
        self.copied = None     # event after the last H2D out of ``host``
        self.cap = ex.capture(stage_images(imgs, ex.device))
        self.copy_stream = None
        self.landing, self.land_free, self.k = [], [None, None], 0

    def run(self, imgs: list) -> PackedBatch:
        src = self.cap.batch.src
        if all(isinstance(i, torch.Tensor) and i.device.type == "cpu" and i.is_pinned() and i.is_contiguous()
               for i in imgs):
            if self.copy_stream is None:
                self.copy_stream = torch.cuda.Stream(device=src.device)
                self.landing = [torch.empty_like(src), torch.empty_like(src)]
                for t in self.landing:  # freed (entry evicted) only once the copy stream is past them
                    t.record_stream(self.copy_stream)
            k, self.k = self.k, self.k ^ 1
            land = self.landing[k]
            compute = torch.cuda.current_stream(src.device)
            with torch.cuda.stream(self.copy_stream):
                if self.land_free[k] is not None:  # the device copy out of this buffer (two calls ago)
                    self.copy_stream.wait_event(self.land_free[k])
                for i, im in enumerate(imgs):
                    land[self.offs[i]:self.offs[i + 1]].copy_(im.view(-1), non_blocking=True)
                landed = torch.cuda.Event()
                landed.record(self.copy_stream)
            compute.wait_event(landed)
            src.copy_(land)
            self.land_free[k] = torch.cuda.Event()
            self.land_free[k].record(compute)
        else:
            if self.host is None:
                self.host = torch.empty(int(self.offs[-1]), dtype=torch.uint8, pin_memory=True)
            if self.copied is not None:
                self.copied.synchronize()  # the previous H2D out of the staging copy has finished
            hv = self.host.numpy()
            for i, im in enumerate(imgs):
                a = im.cpu().numpy() if isinstance(im, torch.Tensor) else im
                hv[self.offs[i]:self.offs[i + 1]] = a.reshape(-1)
            src.copy_(self.host, non_blocking=True)
            self.copied = torch.cuda.Event()
            self.copied.record()
        o = self.cap.replay()
        return PackedBatch(embeds=o.embeds.clone(), tok_offsets=o.tok_offsets.clone(), tiles=list(o.tiles),
                           image_tokens=list(o.image_tokens))


JPEG_DECODE_CHUNK = 32
_DECODE_STREAMS: dict = {}


def _decode_stream(dev: torch.device) -> torch.cuda.Stream:
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _DECODE_STREAMS:
        _DECODE_STREAMS[idx] = torch.cuda.Stream(device=idx)
    return _DECODE_STREAMS[idx]


def stage_jpegs(jpegs, device="cuda") -> ImageBatch:
    """Decode JPEG byte strings on the GPU (nvJPEG via torchvision) straight into one flat device
    buffer of CHW planes; only the compressed bytes cross PCIe."""
    from torchvision.io import ImageReadMode, decode_jpeg
    dev = torch.device(device)
    datas = [j if isinstance(j, torch.Tensor) else torch.frombuffer(bytearray(j), dtype=torch.uint8) for j in jpegs]
    # The decoder runs on its own stream with its own allocator pool: decoding on the compute
    # stream let torchvision's decoder write blocks that the caching allocator had just recycled
    # from tensors still read by in-flight kernels of the previous batch (CUDA error 700 in the
    # back-to-back e2e loop).  The decoded planes are handed to the compute stream by event and
    # record_stream.
    compute = torch.cuda.current_stream(dev)
    dec = _decode_stream(dev)
    imgs = []
    with torch.cuda.stream(dec):
        for i in range(0, len(datas), JPEG_DECODE_CHUNK):
            imgs += decode_jpeg(datas[i:i + JPEG_DECODE_CHUNK], mode=ImageReadMode.RGB, device=dev)
    compute.wait_stream(dec)
    for t in imgs:
        t.record_stream(compute)
    dims = [(int(t.shape[2]), int(t.shape[1])) for t in imgs]
    # no concatenation: K1 reads each decoded image where the decoder left it — src is the image
    # at the lowest address and src_off[i] the byte distance of image i from it
    n = len(imgs)
    if n:
        ptrs = np.array([t.data_ptr() for t in imgs], np.int64)
        base = int(np.argmin(ptrs))
        src = imgs[base]
        offs = ptrs - ptrs[base]
    else:
        src, offs = torch.empty(0, dtype=torch.uint8, device=dev), np.zeros(0, np.int64)
    meta = np.concatenate([offs.view(np.int32), np.array([d[0] for d in dims], np.int32),
                           np.array([d[1] for d in dims], np.int32)])
    dmeta = torch.from_numpy(meta).pin_memory().to(dev, non_blocking=True)
    return ImageBatch(src=src, src_off=dmeta[:2 * n].view(torch.int64), w=dmeta[2 * n:3 * n], h=dmeta[3 * n:4 * n],
                      dims=dims, h2d_bytes=int(sum(d.numel() for d in datas)) + meta.nbytes, chw=True,
                      parts=tuple(imgs))


class ImagePathExecutor:
    """preprocess -> encode -> pack for one model on one GPU (one process per GPU)."""

    # batch shapes (the images' sizes, in order) kept as captured CUDA graphs by encode_images: a
    # shape seen twice is captured, replays then skip the per-kernel launch cost (ViT-B batch 8 is
    # a ~1 ms step of ~120 launches); least recently used shapes are dropped beyond this many
    GRAPH_CACHE_SHAPES = 4

    def __init__(self, spec: ModelSpec, weights: dict | None = None, seed: int = 0, device="cuda",
                 graphs: bool = True, fold_ln: bool | None = None):
        """fold_ln: LayerNorms folded into the GEMMs (default: for encoders with d >= 1024; a narrow
        encoder served at large batches gains from it too).  Fixed per executor, so embeddings
        never depend on the batch an image is encoded in."""
        if spec.encoder is None:
            from ._lib import ProfileError
            raise ProfileError(f"{spec.name}: no encoder configuration; the image path needs one")
        self.spec = spec
        self.device = torch.device(device)
        if weights is None:
            big = param_count(spec) > DEVICE_INIT_PARAMS and self.device.type == "cuda"
            weights = init_weights(spec, seed, device=str(self.device) if big else "cpu")
        self.weights = weights
        self.encoder = DeviceEncoder(spec, self.weights, self.device, fold_ln=fold_ln)
        self.graphs = graphs and self.device.type == "cuda"
        self._graph_cache: OrderedDict = OrderedDict()  # shape -> _GraphEntry
        self._shape_seen: dict = {}

    # ------------------------------------------------------------------ core path
    def encode(self, batch: ImageBatch, out_alloc=None) -> PackedBatch:
        """out_alloc(rows, width) (optional): where the packed output goes (e.g. a slot of the
        LLM-backend GPU's memory, PeerShardChannel.alloc); default a fresh local tensor."""
        spec, enc = self.spec, self.spec.encoder
        n = batch.n
        if n == 0:
            raise SpecError("encode batch must contain at least one image")
        if batch.ready is not None:  # staged on a side stream: order after the copy, keep the memory
            compute = torch.cuda.current_stream(self.device)
            compute.wait_event(batch.ready)
            for t in (batch.src, batch.src_off, batch.w, batch.h, *batch.parts):
                t.record_stream(compute)
        tiles = [tile_count(w, h, spec) for w, h in batch.dims]
        total_tiles = sum(tiles)
        P = (spec.tile_edge_px // enc.patch_px) ** 2
        plan = ops.tile_plan(batch.w, batch.h, spec)
        patches = ops.preprocess(batch.src, batch.src_off, batch.w, batch.h, plan["tile_off"], plan["geom"], n,
                                 total_tiles, spec, self.encoder.k_pad, self.encoder.norm_scale,
                                 self.encoder.norm_shift, chw=batch.chw, src_bytes=batch.src_bytes)
        # attention sequences: all tokens of one image (images never attend to each other)
        S = spec.seq_per_tile  # encoder tokens per tile (patches + class token if any)
        if enc.family == "mllama":  # an image's tiles attend to each other
            seq_len = np.asarray(tiles, np.float64) * S
            cu = ops.seq_offsets(plan["tile_off"], n, S)  # device-side: capturable in a CUDA graph
            n_seq, max_s = n, int(max(tiles)) * S
        else:  # CLIP-family ViTs see every tile alone (multi-tile LLaVA-OV / thumbnails)
            seq_len = np.full(total_tiles, float(S))
            cu = ops.seq_offsets(None, total_tiles, S, device=self.device)
            n_seq, max_s = total_tiles, S
        sum_sq = float(np.sum(seq_len ** 2))
        if enc.family == "mllama":
            tile_image, tile_slot = ops.tile_index(plan["tile_off"], n, total_tiles)
            emb = self.encoder.forward(patches, total_tiles, cu, n_seq, max_s, tile_image, tile_slot, plan["ar_id"],
                                       out_alloc=out_alloc, sum_sq_seqlen=sum_sq)
        else:
            emb = self.encoder.forward(patches, total_tiles, cu, n_seq, max_s, out_alloc=out_alloc,
                                       sum_sq_seqlen=sum_sq)
        return PackedBatch(embeds=emb, tok_offsets=plan["tok_off"], tiles=tiles,
                           image_tokens=[t * spec.tokens_per_tile for t in tiles])

    def capture(self, batch: ImageBatch, out_alloc=None) -> "CapturedEncode":
        """Record ``encode(batch)`` as a CUDA graph (static shapes: same images each replay, or
        new pixels copied into ``batch.src``).  Replay launches the whole path with one call.
        ``out_alloc`` must return the same buffer on every call (e.g. a fixed peer slot)."""
        self.encode(batch, out_alloc=out_alloc)  # first run outside capture: kernel attributes, allocator warm-up
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.encode(batch, out_alloc=out_alloc)
        return CapturedEncode(graph=g, batch=batch, output=out)

    def encode_images(self, images, pinned: bool = True, out_alloc=None) -> PackedBatch:
        """uint8 HWC images (host arrays, or pinned host tensors) -> packed embeddings.  A batch
        shape seen before runs as a replay of its captured graph (``graphs``; not with
        ``out_alloc``, whose destination may change per call)."""
        if not (self.graphs and pinned and out_alloc is None):
            return self.encode(stage_images(images, self.device, pinned), out_alloc=out_alloc)
        imgs = [_as_hwc_u8(i) for i in images]
        key = tuple((int(i.shape[1]), int(i.shape[0])) for i in imgs)
        entry = self._graph_cache.get(key)
        if entry is None:
            seen = self._shape_seen.get(key, 0) + 1
            if len(self._shape_seen) > 4096:
                self._shape_seen.clear()
            self._shape_seen[key] = seen
            if seen < 2 or not imgs:
                return self.encode(stage_images(imgs, self.device, pinned))
            entry = _GraphEntry(self, imgs)
            self._graph_cache[key] = entry
            while len(self._graph_cache) > self.GRAPH_CACHE_SHAPES:
                self._graph_cache.popitem(last=False)
        self._graph_cache.move_to_end(key)
        return entry.run(imgs)

    def encode_jpegs(self, jpegs) -> PackedBatch:
        """JPEG bytes -> GPU decode -> K0..K9 (no host pixel handling at all)."""
        return self.encode(stage_jpegs(jpegs, self.device))

    # ------------------------------------------------------------------ batcher API
    def run(self, batch: list[WorkItem], images: dict, out_alloc=None) -> PackedBatch:
        """Execute one ``form_batch`` result of ENCODE (or PREPROCESS) items.

        images: request_id -> list of uint8 HWC images of that request; each item's
        ``shard_images`` selects its images (reference engine.py:604-625)."""
        if not batch:
            raise SpecError("empty batch")
        flat, spans = [], {}
        for it in batch:
            if it.stage not in (StageKind.ENCODE, StageKind.PREPROCESS):
                raise SpecError(f"item {it.seq}: stage {it.stage.value} is not on the image path")
            req_imgs = images[it.request_id]
            idx = it.shard_images if it.shard_images else tuple(range(len(req_imgs)))
            start = len(flat)
            flat.extend(req_imgs[i] for i in idx)
            spans[it.seq] = (start, len(flat))
        out = self.encode_images(flat, out_alloc=out_alloc)
        out.item_spans = spans
        return out
