"""Modality-aware batcher objects: work items, encode shards and batch formation.

Mirror of the reference engine's batch objects (/root/reference/pkg/src/lmmsim/engine.py):

* ``WorkItem``      engine.py:73-90   (encode items: size_tokens = tiles * tokens_per_tile,
                                      engine.py:613-614; shard_images = image indices)
* ``encode_shard``  engine.py:93-97
* ``form_batch``    engine.py:100-114 scheduler order, one stage per batch, capped by
                                      ``max_batch[stage]`` (default {preprocess: 8, encode: 1},
                                      engine.py:355)

``ImageQueue`` is the B200 build's per-GPU queue in front of ``ImagePathExecutor``: it keeps
the reference's item/batch semantics and adds a real clock.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import policies as pol
from .core import StageKind

DEFAULT_MAX_BATCH = {StageKind.PREPROCESS.value: 8, StageKind.ENCODE.value: 1}


@dataclass
class WorkItem:
    seq: int
    request_id: int
    stage: StageKind
    size_tokens: int
    tiles: int
    enqueue_ms: float
    ttft_slo_ms: float
    text_tokens: int = 0
    image_tokens: int = 0
    shard_images: tuple = ()
    shard_id: int = 0
    deps: set[int] = field(default_factory=set)

    @property
    def runnable(self) -> bool:
        return not self.deps


def encode_shard(images, n_shards: int) -> list[list[int]]:
    """Split a request's images into shards balanced by tile count."""
    if not images:
        return []
    return pol.split_by_tiles([img.tiles for img in images], n_shards)


def form_batch(queue: list[WorkItem], now: float, scheduler: pol.SchedulerKind,
               aging_slo_fraction: float, max_batch: dict) -> list[int]:
    """Queue indices of the next batch: scheduler order, a single stage, at most the cap."""
    order = pol.schedule_order(queue, now, scheduler, aging_slo_fraction)
    if not order:
        return []
    stage = queue[order[0]].stage
    cap = max_batch.get(stage.value, 1)
    picked: list[int] = []
    for idx in order:
        if queue[idx].stage is not stage:
            continue
        picked.append(idx)
        if len(picked) >= cap:
            break
    return picked
