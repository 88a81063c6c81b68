"""Work partitioning: the reference's hybrid CPU/GPU split (hr/scheduler.py)
and its K-way generalisation used to balance buckets / cells over the GPUs
of one box.

``PerfEstimate``/``record_sample``/``current_ratio``/``partition_queue``/
``partition_by_count`` keep the reference's semantics (K = 2 with devices
named CPU/GPU).  ``KWayEstimate`` + ``partition_k`` extend them to K GPUs:
shares proportional to measured speed (inverse time per item), cumulative-sum
cut points, the crossing request joins the earlier device -- for K = 2 the
cut is exactly ``partition_queue``'s.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import MeasurementError

CPU = "CPU"
GPU = "GPU"


@dataclass
class PerfEstimate:
    cpu_time_per_item: float = 0.0
    gpu_time_per_item: float = 0.0
    cpu_samples: int = 0
    gpu_samples: int = 0
    decay: float = 0.0

    def sampled_both(self) -> bool:
        return self.cpu_samples > 0 and self.gpu_samples > 0


def _fold(mean: float, n: int, rate: float, decay: float) -> float:
    if decay > 0.0 and n > 0:
        return mean + decay * (rate - mean)
    return (mean * n + rate) / (n + 1)


def record_sample(est: PerfEstimate, device: str, items: int, elapsed: float) -> PerfEstimate:
    """Running average of time per item (hr/scheduler.py:27-48)."""
    if items < 1 or elapsed <= 0.0:
        raise MeasurementError(f"bad sample: items={items}, elapsed={elapsed}")
    rate = elapsed / items
    if device == CPU:
        est.cpu_time_per_item = _fold(est.cpu_time_per_item, est.cpu_samples, rate, est.decay)
        est.cpu_samples += 1
    elif device == GPU:
        est.gpu_time_per_item = _fold(est.gpu_time_per_item, est.gpu_samples, rate, est.decay)
        est.gpu_samples += 1
    else:
        raise MeasurementError(f"unknown device {device!r}")
    return est


def current_ratio(est: PerfEstimate):
    if not est.sampled_both():
        return 0.5, 0.5
    a, b = 1.0 / est.cpu_time_per_item, 1.0 / est.gpu_time_per_item
    return a / (a + b), b / (a + b)


@dataclass
class Partition:
    cpu_set: list
    gpu_set: list
    cpu_target_items: float
    crossing_items: int = 0


def _cut(weights, target: float, nearest: bool):
    """Shortest prefix whose cumulative weight reaches target (the crossing
    element included unless `nearest` lands closer without it)."""
    cum = 0.0
    for i, w in enumerate(weights):
        cum += w
        if cum >= target:
            if nearest and (cum - target) > (target - (cum - w)):
                return i, w
            return i + 1, w
    return len(weights), (weights[-1] if weights else 0)


def partition_queue(queue, est: PerfEstimate, cpu_share: float | None = None, nearest_target: bool = False):
    """hr/scheduler.py:73-107"""
    if cpu_share is None:
        cpu_share, _ = current_ratio(est)
    total = sum(w.item_count for w in queue)
    target = total * cpu_share
    if not queue or target <= 0.0:
        return Partition([], list(queue), target)
    k, crossing = _cut([w.item_count for w in queue], target, nearest_target)
    return Partition(list(queue[:k]), list(queue[k:]), target, crossing)


def partition_by_count(queue, cpu_fraction: float):
    k = int(len(queue) * cpu_fraction)
    return Partition(list(queue[:k]), list(queue[k:]), 0.0)


@dataclass
class KWayEstimate:
    """Per-device running time per item for K devices."""

    k: int
    time_per_item: list = field(default_factory=list)
    samples: list = field(default_factory=list)
    decay: float = 0.0

    def __post_init__(self):
        if not self.time_per_item:
            self.time_per_item = [0.0] * self.k
            self.samples = [0] * self.k

    def record(self, device: int, items: int, elapsed: float):
        if items < 1 or elapsed <= 0.0:
            raise MeasurementError(f"bad sample: items={items}, elapsed={elapsed}")
        self.time_per_item[device] = _fold(self.time_per_item[device], self.samples[device], elapsed / items,
                                           self.decay)
        self.samples[device] += 1

    def shares(self):
        """Speed-proportional shares; equal until every device has a sample."""
        if not all(self.samples):
            return [1.0 / self.k] * self.k
        speed = [1.0 / t for t in self.time_per_item]
        s = sum(speed)
        return [v / s for v in speed]


def partition_k(weights, shares, nearest_target: bool = False):
    """Cut a weighted sequence into len(shares) contiguous ranges; returns the
    K+1 boundaries.  Device d's target is the cumulative share up to d; each
    crossing element stays with the earlier device (as partition_queue)."""
    total = float(sum(weights))
    bounds = [0]
    start = 0
    acc_share = 0.0
    for d, sh in enumerate(shares[:-1]):
        acc_share += sh
        target = total * acc_share - sum(weights[:start])
        if start >= len(weights) or target <= 0.0:
            bounds.append(start)
            continue
        k, _ = _cut(weights[start:], target, nearest_target)
        start += k
        bounds.append(start)
    bounds.append(len(weights))
    return bounds
