"""Synthetic image-request source and trace I/O for the image path.

Restates the reference workload generator (/root/reference/pkg/src/lmmsim/workload.py) draw
for draw, so a given (config, seed) yields the same requests, image sizes and tile counts:

* ``GeneratorConfig`` / ``BurstEpisode``   workload.py:124-178
* ``DEFAULT_IMAGES_PER_REQUEST``           workload.py:140
* ``sample_power_law``                     workload.py:181-185
* rate segments                            workload.py:199-219
* ``generate``                             workload.py:222-296 (image dims: :247-252)
* trace cell parsing / ``load_trace``      workload.py:43-108, ``write_trace`` :111-121

Pinned against the reference by tests/golden/generator_*.json (made by
tests/golden/make_golden.py, which imports the reference in the authoring container).
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .core import ImageSpec, ModelSpec, Request


class TraceError(ValueError):
    """Unreadable or badly malformed trace file."""


TRACE_COLUMNS = ["arrival_ms", "service_id", "text_tokens", "num_images", "image_dims", "output_tokens"]

DEFAULT_IMAGES_PER_REQUEST = {1: 0.55, 2: 0.20, 3: 0.08, 4: 0.06, 5: 0.04, 6: 0.03, 8: 0.02, 12: 0.01,
                              16: 0.01}


@dataclass(frozen=True)
class BurstEpisode:
    start_ms: float
    duration_ms: float
    rate_multiplier: float = 1.0
    image_multiplier: float = 1.0

    @property
    def end_ms(self) -> float:
        return self.start_ms + self.duration_ms


@dataclass
class GeneratorConfig:
    model: ModelSpec
    base_rate: float = 5.0
    burst_episodes: tuple[BurstEpisode, ...] = ()
    text_len_alpha: float = 2.9
    image_req_len_alpha: float = 4.4
    text_len_min: int = 16
    text_len_max: int = 32768
    image_req_len_min: int = 16
    image_req_len_max: int = 32768
    image_request_fraction: float = 0.3
    images_per_request: dict[int, float] = field(default_factory=lambda: dict(DEFAULT_IMAGES_PER_REQUEST))
    image_dim_median_px: float = 500.0
    image_dim_sigma: float = 0.55
    image_dim_min_px: int = 64
    image_dim_max_px: int = 4096
    output_len_median: int = 128
    output_len_sigma: float = 0.7
    output_len_max: int = 2048
    seed: int = 0

    def validate(self) -> None:
        if self.base_rate <= 0:
            raise ValueError("base_rate must be > 0")
        if not 0.0 <= self.image_request_fraction <= 1.0:
            raise ValueError("image_request_fraction must be in [0, 1]")
        if self.text_len_alpha <= 1 or self.image_req_len_alpha <= 1:
            raise ValueError("power-law exponents must be > 1")
        total = sum(self.images_per_request.values())
        if abs(total - 1.0) > 1e-6:
            raise ValueError(f"images_per_request probabilities sum to {total}, expected 1")
        if any(k < 1 or k > 16 for k in self.images_per_request):
            raise ValueError("images_per_request keys must be in 1..16")


def sample_power_law(rng: np.random.Generator, alpha: float, lo: int, hi: int, size=None):
    """Pareto draw with density exponent ``alpha`` clamped to [lo, hi]."""
    u = rng.random(size)
    return np.clip(lo * u ** (-1.0 / (alpha - 1.0)), lo, hi)


def _segments(cfg: GeneratorConfig, horizon_ms: float):
    cuts = {0.0, horizon_ms}
    for ep in cfg.burst_episodes:
        cuts.add(min(max(ep.start_ms, 0.0), horizon_ms))
        cuts.add(min(max(ep.end_ms, 0.0), horizon_ms))
    pts = sorted(cuts)
    for lo, hi in zip(pts, pts[1:]):
        if hi <= lo:
            continue
        mid = 0.5 * (lo + hi)
        rate_mult = img_mult = 1.0
        for ep in cfg.burst_episodes:
            if ep.start_ms <= mid < ep.end_ms:
                rate_mult *= ep.rate_multiplier
                img_mult *= ep.image_multiplier
        yield lo, hi, rate_mult, img_mult


def _lognormal_dim(rng, cfg: GeneratorConfig) -> int:
    return int(np.clip(cfg.image_dim_median_px * math.exp(rng.normal(0.0, cfg.image_dim_sigma)),
                       cfg.image_dim_min_px, cfg.image_dim_max_px))


def generate(cfg: GeneratorConfig, horizon_ms: float) -> list[Request]:
    """Request stream over [0, horizon_ms), identical to the reference for the same seed."""
    if horizon_ms <= 0:
        raise ValueError("horizon_ms must be > 0")
    cfg.validate()
    rng = np.random.default_rng(cfg.seed)
    counts = sorted(cfg.images_per_request)
    probs = np.array([cfg.images_per_request[k] for k in counts])
    probs = probs / probs.sum()
    out: list[Request] = []
    for seg_lo, seg_hi, rate_mult, img_mult in _segments(cfg, horizon_ms):
        mean_gap = 1.0 / (cfg.base_rate * rate_mult / 1000.0)
        t = seg_lo
        while True:
            t += rng.exponential(mean_gap)
            if t >= seg_hi:
                break
            if rng.random() < cfg.image_request_fraction:
                n_img = int(counts[rng.choice(len(counts), p=probs)])
                if img_mult != 1.0:
                    n_img = min(16, max(1, int(round(n_img * img_mult))))
                images = []
                for _ in range(n_img):
                    w = _lognormal_dim(rng, cfg)
                    h = _lognormal_dim(rng, cfg)
                    images.append(ImageSpec.from_dims(w, h, cfg.model))
                total = float(sample_power_law(rng, cfg.image_req_len_alpha, cfg.image_req_len_min,
                                               cfg.image_req_len_max))
                text = max(cfg.text_len_min, int(round(total)) - sum(i.image_tokens for i in images))
                service = "video" if n_img >= 8 else "vision"
            else:
                images = []
                text = int(round(float(sample_power_law(rng, cfg.text_len_alpha, cfg.text_len_min,
                                                        cfg.text_len_max))))
                service = "chat"
            n_out = int(np.clip(cfg.output_len_median * math.exp(rng.normal(0.0, cfg.output_len_sigma)),
                                1, cfg.output_len_max))
            out.append(Request(id=len(out), arrival_ms=t, text_tokens=text, images=tuple(images),
                               output_tokens=n_out, service_id=service))
    return out


def image_dims_of(requests: list[Request]) -> list[tuple[int, int]]:
    return [(i.width_px, i.height_px) for r in requests for i in r.images]


def parse_dims(cell: str) -> list[tuple[int, int]]:
    """``"WxH;WxH"`` trace cell -> [(w, h)] (reference workload.py:43-51)."""
    cell = cell.strip()
    if not cell:
        return []
    dims = []
    for part in cell.split(";"):
        w, h = part.lower().split("x")
        dims.append((int(w), int(h)))
    return dims


@dataclass
class TraceRecord:
    """One parsed trace row (reference workload.py:28-33)."""
    arrival_ms: float
    service_id: str
    text_tokens: int
    image_dims: list[tuple[int, int]]
    output_tokens: int


@dataclass
class TraceLoadResult:
    """``load_trace`` result (reference workload.py:36-40)."""
    requests: list[Request]
    malformed_rows: int
    total_rows: int


def load_trace(path: str | Path, model: ModelSpec, max_malformed_frac: float = 0.01) -> TraceLoadResult:
    """Trace CSV -> requests sorted by arrival (reference workload.py:54-108).

    Malformed rows are counted and skipped; a malformed share above ``max_malformed_frac``
    raises ``TraceError``. Requests get ids 0..n-1 in arrival order.
    """
    path = Path(path)
    if not path.exists():
        raise TraceError(f"trace file not found: {path}")
    records: list[TraceRecord] = []
    bad = total = 0
    with path.open(newline="") as fh:
        reader = csv.DictReader(fh)
        if reader.fieldnames is None:
            return TraceLoadResult([], 0, 0)
        missing = [c for c in TRACE_COLUMNS if c not in reader.fieldnames]
        if missing:
            raise TraceError(f"trace {path} missing columns: {missing}")
        for row in reader:
            total += 1
            try:
                dims = parse_dims(row["image_dims"] or "")
                if int(row["num_images"]) != len(dims):
                    raise ValueError("num_images does not match image_dims")
                rec = TraceRecord(arrival_ms=float(row["arrival_ms"]),
                                  service_id=row["service_id"] or "default",
                                  text_tokens=int(row["text_tokens"]), image_dims=dims,
                                  output_tokens=int(row["output_tokens"]))
                if rec.arrival_ms < 0 or rec.text_tokens < 0 or rec.output_tokens < 1:
                    raise ValueError("negative counts")
                records.append(rec)
            except (ValueError, KeyError):
                bad += 1
    if total and bad / total > max_malformed_frac:
        raise TraceError(f"{bad}/{total} malformed rows in {path} exceeds {max_malformed_frac:.0%}")
    records.sort(key=lambda r: r.arrival_ms)
    reqs = [Request(id=i, arrival_ms=r.arrival_ms, text_tokens=r.text_tokens,
                    output_tokens=r.output_tokens, service_id=r.service_id,
                    images=tuple(ImageSpec.from_dims(w, h, model) for w, h in r.image_dims))
            for i, r in enumerate(records)]
    return TraceLoadResult(reqs, bad, total)


def write_trace(path: str | Path, requests: list[Request]) -> None:
    """Requests -> trace CSV, the inverse of ``load_trace`` (reference workload.py:111-121)."""
    with Path(path).open("w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(TRACE_COLUMNS)
        for r in requests:
            wr.writerow([f"{r.arrival_ms:.3f}", r.service_id, r.text_tokens, len(r.images),
                         ";".join(f"{i.width_px}x{i.height_px}" for i in r.images), r.output_tokens])
