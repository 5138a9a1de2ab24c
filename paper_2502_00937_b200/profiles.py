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
profile keys on the batch's total tiles measured with the generator's tile mix and
interpolates piecewise-linearly between measured points.
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

    def encode_ms_per_tile(self) -> float:
        """Marginal ms per tile at the largest measured batch (throughput regime)."""
        t, ms = self.encode_points[-1]
        return ms / t

    # ---------------------------------------------------------------- serialisation
    def to_dict(self) -> dict:
        return {"model": self.model.name, "encode_points": [list(p) for p in self.encode_points],
                "preprocess_ms_per_tile": self.preprocess_ms_per_tile,
                "preprocess_floor_ms": self.preprocess_floor_ms, "measured_tp": list(self.measured_tp),
                "meta": self.meta}

    @classmethod
    def from_dict(cls, d: dict, model: ModelSpec) -> "MeasuredProfile":
        if d["model"] != model.name:
            raise ProfileError(f"profile is for {d['model']}, not {model.name}")
        return cls(model=model, encode_points=[tuple(p) for p in d["encode_points"]],
                   preprocess_ms_per_tile=float(d["preprocess_ms_per_tile"]),
                   preprocess_floor_ms=float(d.get("preprocess_floor_ms", 0.0)),
                   measured_tp=tuple(d.get("measured_tp", (1,))), meta=dict(d.get("meta", {})))

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_dict(), indent=2) + "\n")

    def to_reference_profile(self, base: dict, cpu_cores: int | None = None) -> dict:
        """Merge measured image-stage constants into a reference profile dict (the output of
        ``lmmsim calibrate``, schema profiles.py:268-293): the LLM-side fields are kept, the
        image-stage fields are replaced by B200 measurements.

        ``prep_ms_per_tile_core`` is the per-tile cost times the core count the reference divides
        by (so ``preprocess_latency`` returns the measured GPU time for that core count);
        ``encode_ms_per_tile`` holds the measured marginal ms per tile for each measured TP."""
        if base.get("model") != self.model.name:
            raise ProfileError(f"base profile is for {base.get('model')}, not {self.model.name}")
        out = dict(base)
        cores = cpu_cores or int(base.get("ref_cpu_cores", 8))
        out["prep_ms_per_tile_core"] = self.preprocess_ms_per_tile * cores
        out["prep_floor_ms"] = self.preprocess_floor_ms
        out["encode_ms_per_tile"] = {str(tp): self.encode_ms_per_tile() for tp in self.measured_tp}
        return out


def measure_profile(executor, batch_sizes=(1, 4, 16, 32), warmup: int = 2, iters: int = 5,
                    seed: int = 0) -> MeasuredProfile:
    """Time the real image path (CUDA events) on generator-drawn images at several batch
    sizes; returns the measured profile.  Needs a GPU."""
    import numpy as np
    import torch

    from . import ops, workload
    from .core import tile_count
    from .executor import stage_images

    spec = executor.spec
    cfg = workload.GeneratorConfig(model=spec, base_rate=50.0, image_request_fraction=1.0, seed=seed)
    dims = workload.image_dims_of(workload.generate(cfg, 20_000.0))
    rng = np.random.default_rng(seed)
    points, prep = [], []
    for b in batch_sizes:
        d = dims[:b]
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
        tiles = sum(tile_count(w, h, spec) for w, h in d)
        points.append((tiles, s.elapsed_time(e) / iters))
        k = log.summary()
        prep_ms = sum(k.get(n, {}).get("ms", 0.0) for n in ("tile_plan", "preprocess")) / iters
        prep.append(prep_ms / tiles)
    return MeasuredProfile(model=spec, encode_points=points, preprocess_ms_per_tile=float(np.mean(prep)),
                           meta={"device": torch.cuda.get_device_name(), "batch_sizes": list(batch_sizes),
                                 "iters": iters, "tile_mix": "reference generator, seed %d" % seed})
