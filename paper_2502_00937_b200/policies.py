"""Image routing and batch ordering: the data-parallel partition of images over GPUs.

Mirror of the image-path parts of the reference policy library
(/root/reference/pkg/src/lmmsim/policies.py):

* ``split_by_tiles``  policies.py:91-101   greedy largest-first partition by tile count
* ``route_image``     policies.py:104-124  fanout = min(#images, #instances, max_fanout)
* ``schedule_order``  policies.py:153-173  FIFO / SLO-priority with aging
* ``schedule_next``   policies.py:176-179

``split_by_cost`` is the B200 build's performance-mode partition: the same greedy rule
weighted by each image's encoder FLOPs (attention cost is super-linear in tiles, so tile
counts under-weight large images).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


class RouterKind(str, Enum):
    ROUND_ROBIN = "round_robin"
    LEAST_PENDING = "least_pending"


class SchedulerKind(str, Enum):
    FIFO = "fifo"
    SLO_PRIORITY = "slo_priority"


@dataclass(frozen=True)
class PolicySet:
    """Image-path subset of the reference PolicySet (policies.py:48-62)."""

    router: RouterKind = RouterKind.LEAST_PENDING
    scheduler: SchedulerKind = SchedulerKind.SLO_PRIORITY
    max_fanout: int = 8
    aging_slo_fraction: float = 0.5


def _greedy_partition(weights, n_shards: int) -> list[list[int]]:
    n = max(1, min(n_shards, len(weights)))
    load = [0] * n
    shards: list[list[int]] = [[] for _ in range(n)]
    # heaviest first, ties by index; each goes to the least-loaded shard (ties: lowest shard)
    for idx in sorted(range(len(weights)), key=lambda i: (-weights[i], i)):
        target = min(range(n), key=lambda s: (load[s], s))
        shards[target].append(idx)
        load[target] += weights[idx]
    return [sorted(s) for s in shards if s]


def split_by_tiles(tile_sizes: list[int], n_shards: int) -> list[list[int]]:
    """Greedy largest-first partition of image indices balanced by tile count."""
    return _greedy_partition(list(tile_sizes), n_shards)


def split_by_cost(costs: list[float], n_shards: int) -> list[list[int]]:
    """Same greedy rule, weighted by per-image cost (e.g. encoder FLOPs)."""
    return _greedy_partition(list(costs), n_shards)


def route_image(request, instances, router: RouterKind, max_fanout: int, rr_state: dict):
    """Assign a request's images to image instances -> [(instance, [image indices])].

    Least-pending takes the ``fanout`` instances with the fewest pending image tokens
    (ties: lowest id); round-robin walks the id-sorted pool from a persistent cursor.
    """
    if not instances:
        return None
    tiles = [img.tiles for img in request.images]
    fanout = min(len(tiles), len(instances), max_fanout)
    if router == RouterKind.ROUND_ROBIN:  # by value: the reference's own enum members work too
        pool = sorted(instances, key=lambda inst: inst.id)
        start = rr_state.get("image", 0)
        rr_state["image"] = start + fanout
        chosen = [pool[(start + k) % len(pool)] for k in range(fanout)]
    else:
        chosen = sorted(instances, key=lambda inst: (inst.pending_image_tokens, inst.id))[:fanout]
    return list(zip(chosen, split_by_tiles(tiles, len(chosen))))


def schedule_order(items, now: float, scheduler: SchedulerKind, aging_slo_fraction: float):
    """Runnable queue indices in execution order.

    SLO-priority runs the smallest item first, except that items waiting longer than
    ``aging_slo_fraction`` of their TTFT SLO go first in FIFO order (starvation bound).
    """
    runnable = [i for i, it in enumerate(items) if it.runnable]
    fifo_key = lambda i: (items[i].enqueue_ms, items[i].seq)  # noqa: E731
    if scheduler == SchedulerKind.FIFO:
        return sorted(runnable, key=fifo_key)
    aged = [i for i in runnable if now - items[i].enqueue_ms > aging_slo_fraction * items[i].ttft_slo_ms]
    aged_set = set(aged)
    fresh = [i for i in runnable if i not in aged_set]
    aged.sort(key=fifo_key)
    fresh.sort(key=lambda i: (items[i].size_tokens, items[i].enqueue_ms, items[i].seq))
    return aged + fresh


def schedule_next(items, now: float, scheduler: SchedulerKind, aging_slo_fraction: float = 0.5):
    order = schedule_order(items, now, scheduler, aging_slo_fraction)
    return order[0] if order else None
