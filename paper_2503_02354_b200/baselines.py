"""Comparison policies behind the same evictor / assigner seams.

Mirror of ``coesim.baselines`` (``/root/reference/pkg/src/coesim/baselines.py``):
LRU (recency advances on every load and batch, baselines.py:20-34), FIFO
(only an absent->resident transition stamps, baselines.py:37-51), the shared
prefix eviction over a stamp order (baselines.py:54-73) and round-robin
assignment (baselines.py:76-88).  Needed for the ``samba_*`` and ablation
policies the xLRU / switch-reduction figures are measured against.
"""

from __future__ import annotations

from itertools import count
from typing import Iterable

from .types import MemoryStarvationError


def _evict_in_order(pool, needed_bytes: int, key) -> list:
    deficit = needed_bytes - pool.free_bytes
    if deficit <= 0:
        return []
    order = sorted((eid for eid in pool.resident if eid not in pool.pinned), key=lambda eid: (key(eid), eid))
    victims, reclaimed = [], 0.0
    for eid in order:
        if reclaimed >= deficit:
            break
        victims.append(eid)
        reclaimed += pool.resident[eid]
    if reclaimed < deficit:
        raise MemoryStarvationError(
            f"pool {pool.executor_id}: evicting every unpinned expert frees {reclaimed} bytes, "
            f"still short of {deficit}")
    return victims


class _StampedEvictor:
    def __init__(self) -> None:
        self._ticks = count()
        self._stamps: dict = {}

    def _stamp(self, expert_id: str) -> None:
        self._stamps[expert_id] = next(self._ticks)

    def select(self, pool, needed_bytes: int, pending_targets: Iterable[str] = ()) -> list:
        return _evict_in_order(pool, needed_bytes, key=lambda eid: self._stamps.get(eid, -1))


class LruEvictor(_StampedEvictor):
    """Least-recently-executed first; ``touch`` on every load and batch."""

    def touch(self, expert_id: str) -> None:
        self._stamp(expert_id)


class FifoEvictor(_StampedEvictor):
    """Residency-arrival order; ``on_resident`` only on absent->resident."""

    def on_resident(self, expert_id: str) -> None:
        self._stamp(expert_id)


class RoundRobinAssigner:
    """Executors in id order, one request each."""

    def __init__(self, num_executors: int):
        if num_executors < 1:
            raise ValueError("need at least one executor")
        self.num_executors = num_executors
        self._cursor = 0

    def next_executor(self) -> int:
        chosen = self._cursor
        self._cursor = (chosen + 1) % self.num_executors
        return chosen
