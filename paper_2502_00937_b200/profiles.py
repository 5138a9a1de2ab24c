"""Measured-latency profile: B200 numbers behind the reference's stage-latency seam.

The reference simulator consumes a ``LatencyProfile`` whose two image-path methods are
``preprocess_latency(tiles, cpu_cores)`` (profiles.py:128-134) and
``encode_latency(batch_tiles, tp)`` (profiles.py:136-145), both modelled analytically from
TTFT shares.  ``MeasuredProfile`` exposes the same two methods with the same argument meaning
and error behaviour (``ProfileError`` for an empty batch or an unmeasured TP degree), backed by
timings of the real image path on a B200 (``measure_profile``), and exports them into the
reference's profile JSON schema (profiles.py:268-293) so that ``lmmsim`` autoscaling and
capacity planning can run on measured numbers.

Encode cost is not linear in tiles (attention is quadratic in an image's tokens), so the
profile keeps two measurements: the batch's total tiles with the generator's tile mix
(piecewise-linear, behind the reference's ``encode_latency(batch_tiles, tp)``), and the cost of
an image of each tile count inside a full batch (``encode_latency_images``: a batch priced from
its tile histogram).

TP: the B200 build scales the encoder by data parallelism over images (north_star), not by
tensor parallelism.  ``measured_tp`` lists the degrees whose latency is known; the export to
the reference schema writes, for each TP degree of the spec, the DP-equivalent latency — the
batch split over that many GPUs (``dp_efficiency`` = measured multi-GPU throughput over N x the
one-GPU throughput, 1.0 when unmeasured) — so a reference simulation whose ``select_sharding``
picks TP > 1 prices it with what that many B200s achieve on this path.
"""

from __future__ import annotations

import bisect
import json
from dataclasses import dataclass, field
from pathlib import Path

from .core import ModelSpec


class ProfileError(ValueError):
    """Bad inputs to a latency model (same role as lmmsim.profiles.ProfileError)."""


@dataclass
class MeasuredProfile:
    model: ModelSpec
    encode_points: list[tuple[int, float]]          # (batch tiles, ms), sorted by tiles
    preprocess_ms_per_tile: float                   # GPU preprocessing (K0 + K1) per tile
    preprocess_floor_ms: float = 0.0
    measured_tp: tuple[int, ...] = (1,)
    meta: dict = field(default_factory=dict)
    tile_costs: dict = field(default_factory=dict)  # tiles per image -> ms per image inside a batch
    dp_efficiency: dict = field(default_factory=dict)  # GPUs -> throughput / (GPUs x one-GPU throughput)

    def __post_init__(self):
        self.encode_points = sorted((int(t), float(ms)) for t, ms in self.encode_points)
        if not self.encode_points:
            raise ProfileError("measured profile needs at least one encode point")

    # ---------------------------------------------------------------- reference seam
    def preprocess_latency(self, tiles: int, cpu_cores: int) -> float:
        """Preprocessing time of a batch.  On this build preprocessing runs on the GPU (K1), so
        host cores do not scale it; the argument is validated like the reference's."""
        if cpu_cores < 1:
            raise ProfileError("cpu_cores must be >= 1")
        if tiles <= 0:
            return 0.0
        return max(self.preprocess_floor_ms, self.preprocess_ms_per_tile * tiles)

    def encode_latency(self, batch_tiles: int, tp: int) -> float:
        """Measured encode time of a batch with ``batch_tiles`` tiles (piecewise linear)."""
        if batch_tiles < 1:
            raise ProfileError("encode batch must contain at least one tile")
        if tp not in self.model.supported_tp_encoder or tp not in self.measured_tp:
            raise ProfileError(f"TP-{tp} not measured for {self.model.name} encoder "
                               f"(measured: {sorted(self.measured_tp)})")
        pts = self.encode_points
        xs = [p[0] for p in pts]
        if len(pts) == 1:
            return pts[0][1] * batch_tiles / pts[0][0]
        i = bisect.bisect_left(xs, batch_tiles)
        if i < len(xs) and xs[i] == batch_tiles:
            return pts[i][1]
        lo, hi = (pts[0], pts[1]) if i == 0 else (pts[-2], pts[-1]) if i >= len(pts) else (pts[i - 1], pts[i])
        slope = (hi[1] - lo[1]) / (hi[0] - lo[0])
        return max(0.0, lo[1] + slope * (batch_tiles - lo[0]))

    def encode_latency_images(self, tiles_list, tp: int = 1) -> float:
        """Measured encode time of a batch priced from its tile histogram (ms): sum over images of
        the per-image cost of its tile count (super-linear in tiles), over ``tp`` DP GPUs."""
        if not tiles_list:
            raise ProfileError("encode batch must contain at least one image")
        if not self.tile_costs:
            return self.encode_latency(int(sum(tiles_list)), tp)
        if tp not in self.dp_gpus():
            raise ProfileError(f"{tp} GPUs not measured for {self.model.name} (measured: {self.dp_gpus()})")
        costs = {int(k): float(v) for k, v in self.tile_costs.items()}
        known = sorted(costs)
        total = 0.0
        for t in tiles_list:
            if t in costs:
                total += costs[t]
            else:  # nearest measured tile count, scaled quadratically in tokens
                k = min(known, key=lambda u: abs(u - t))
                total += costs[k] * (t / k) ** 2
        return total / (tp * self.dp_efficiency.get(tp, 1.0))

    def dp_gpus(self) -> list[int]:
        return sorted({1, *(int(k) for k in self.dp_efficiency)})

    def encode_ms_per_tile(self) -> float:
        """Marginal ms per tile at the largest measured batch (throughput regime)."""
        t, ms = self.encode_points[-1]
        return ms / t

    # ---------------------------------------------------------------- serialisation
    def to_dict(self) -> dict:
        return {"model": self.model.name, "encode_points": [list(p) for p in self.encode_points],
                "preprocess_ms_per_tile": self.preprocess_ms_per_tile,
                "preprocess_floor_ms": self.preprocess_floor_ms, "measured_tp": list(self.measured_tp),
                "tile_costs": {str(k): v for k, v in self.tile_costs.items()},
                "dp_efficiency": {str(k): v for k, v in self.dp_efficiency.items()},
                "meta": self.meta}

    @classmethod
    def from_dict(cls, d: dict, model: ModelSpec) -> "MeasuredProfile":
        if d["model"] != model.name:
            raise ProfileError(f"profile is for {d['model']}, not {model.name}")
        return cls(model=model, encode_points=[tuple(p) for p in d["encode_points"]],
                   preprocess_ms_per_tile=float(d["preprocess_ms_per_tile"]),
                   preprocess_floor_ms=float(d.get("preprocess_floor_ms", 0.0)),
                   measured_tp=tuple(d.get("measured_tp", (1,))), meta=dict(d.get("meta", {})),
                   tile_costs={int(k): float(v) for k, v in d.get("tile_costs", {}).items()},
                   dp_efficiency={int(k): float(v) for k, v in d.get("dp_efficiency", {}).items()})

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_dict(), indent=2) + "\n")

    def to_reference_profile(self, base: dict, cpu_cores: int | None = None) -> dict:
        """Merge measured image-stage constants into a reference profile dict (the output of
        ``lmmsim calibrate``, schema profiles.py:268-293): the LLM-side fields are kept, the
        image-stage fields are replaced by B200 measurements.

        ``prep_ms_per_tile_core`` is the per-tile cost times the core count the reference divides
        by (so ``preprocess_latency`` returns the measured GPU time for that core count);
        ``encode_ms_per_tile`` holds the measured marginal ms per tile for every TP degree the
        spec supports, TP > 1 as its DP-equivalent (ms per tile / (tp x dp_efficiency[tp]))."""
        if base.get("model") != self.model.name:
            raise ProfileError(f"base profile is for {base.get('model')}, not {self.model.name}")
        out = dict(base)
        cores = cpu_cores or int(base.get("ref_cpu_cores", 8))
        out["prep_ms_per_tile_core"] = self.preprocess_ms_per_tile * cores
        out["prep_floor_ms"] = self.preprocess_floor_ms
        m = self.encode_ms_per_tile()
        out["encode_ms_per_tile"] = {str(tp): m / (tp * self.dp_efficiency.get(tp, 1.0))
                                     for tp in self.model.supported_tp_encoder}
        out["b200_measured"] = {"encode_points": [list(p) for p in self.encode_points],
                                "tile_costs": {str(k): v for k, v in self.tile_costs.items()},
                                "tp_semantics": "TP>1 = data parallel over that many B200s (DP-equivalent)",
                                "dp_efficiency": {str(k): v for k, v in self.dp_efficiency.items()}}
        return out


def measure_profile(executor, batch_sizes=(1, 4, 16, 32), warmup: int = 2, iters: int = 5,
                    seed: int = 0, per_count_batch: int = 8) -> MeasuredProfile:
    """Time the real image path (CUDA events) on generator-drawn images at several batch sizes,
    and the per-image cost of every tile count inside a batch of ``per_count_batch`` images of
    that count; returns the measured profile.  Needs a GPU."""
    import numpy as np
    import torch

    from . import ops, workload
    from .core import tile_count
    from .executor import stage_images

    spec = executor.spec
    cfg = workload.GeneratorConfig(model=spec, base_rate=50.0, image_request_fraction=1.0, seed=seed)
    dims = workload.image_dims_of(workload.generate(cfg, 20_000.0))
    rng = np.random.default_rng(seed)

    def time_batch(d):
        imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in d]
        staged = stage_images(imgs, executor.device)
        for _ in range(warmup):
            executor.encode(staged)
        log = ops.LaunchLog(timing=True)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ops.LOG = log
        s.record()
        for _ in range(iters):
            executor.encode(staged)
        e.record()
        ops.LOG = None
        torch.cuda.synchronize()
        k = log.summary()
        prep_ms = sum(k.get(n, {}).get("ms", 0.0) for n in ("tile_plan", "preprocess")) / iters
        return s.elapsed_time(e) / iters, prep_ms

    points, prep = [], []
    for b in batch_sizes:
        d = dims[:b]
        ms, prep_ms = time_batch(d)
        tiles = sum(tile_count(w, h, spec) for w, h in d)
        points.append((tiles, ms))
        prep.append(prep_ms / tiles)
    tile_costs = {}
    by_count: dict = {}
    for w, h in dims:
        by_count.setdefault(tile_count(w, h, spec), []).append((w, h))
    for t in sorted(by_count):
        d = (by_count[t] * per_count_batch)[:per_count_batch]
        ms, _ = time_batch(d)
        tile_costs[t] = ms / len(d)
    return MeasuredProfile(model=spec, encode_points=points, preprocess_ms_per_tile=float(np.mean(prep)),
                           tile_costs=tile_costs,
                           meta={"device": torch.cuda.get_device_name(), "batch_sizes": list(batch_sizes),
                                 "per_count_batch": per_count_batch, "iters": iters,
                                 "tile_mix": "reference generator, seed %d" % seed})
