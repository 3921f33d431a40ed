"""Value types of the mapping/migration path, interface-compatible with the
reference's `spotsim.domain` (domain.py:37-296).

The hot-path functions in this package duck-type their inputs, so they
accept either these classes or the reference's own; results are built with
the caller's classes (see `_types.result_types`).  These definitions make the
package usable standalone (no reference installed).
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass, field
from fractions import Fraction

GpuRef = tuple[str, int]
Interval = tuple[Fraction, Fraction]


class DomainError(ValueError):
    """Invalid domain value (reference: domain.py:27-28)."""


_DIGITS = re.compile(r"(\d+)")


def natural_key(instance_id: str):
    """'i-2' sorts before 'i-10' (reference: domain.py:31-34)."""
    return tuple(int(t) if t.isdigit() else t for t in _DIGITS.split(instance_id))


@dataclass(frozen=True, order=True)
class ParallelConfig:
    """(D, P, M) plus batch cap (reference: domain.py:37-71)."""

    data_parallel: int
    pipeline_stages: int
    tensor_shards: int
    batch_limit: int

    def __post_init__(self):
        for name in ("data_parallel", "pipeline_stages", "tensor_shards", "batch_limit"):
            if getattr(self, name) < 1:
                raise DomainError(f"{name} must be >= 1, got {getattr(self, name)}")

    @property
    def gpus(self) -> int:
        return self.data_parallel * self.pipeline_stages * self.tensor_shards

    @property
    def concurrent_requests(self) -> int:
        return self.data_parallel * self.batch_limit

    def instances(self, gpus_per_instance: int) -> int:
        return math.ceil(self.gpus / gpus_per_instance)

    def as_tuple(self):
        return (self.data_parallel, self.pipeline_stages, self.tensor_shards, self.batch_limit)

    def shape(self):
        return (self.data_parallel, self.pipeline_stages, self.tensor_shards)


@dataclass(frozen=True, order=True)
class TopologyPosition:
    """1-based (pipeline, stage, shard) (reference: domain.py:74-89)."""

    pipeline: int
    stage: int
    shard: int


def positions(config) -> list:
    """Lexicographic (d, p, m) order (reference: domain.py:92-99)."""
    D, P, M = config.data_parallel, config.pipeline_stages, config.tensor_shards
    return [TopologyPosition(d, p, m) for d in range(1, D + 1) for p in range(1, P + 1)
            for m in range(1, M + 1)]


@dataclass(frozen=True)
class ModelSpec:
    """Uniform per-layer memory geometry (reference: domain.py:102-117)."""

    name: str
    num_layers: int
    bytes_per_layer: int
    kv_bytes_per_token_per_layer: int

    def __post_init__(self):
        if self.num_layers < 1 or self.bytes_per_layer <= 0:
            raise DomainError("model must have >=1 layers with positive bytes")

    @property
    def total_param_bytes(self) -> int:
        return self.num_layers * self.bytes_per_layer


@dataclass
class RequestSpec:
    """(reference: domain.py:120-136)"""

    id: str
    arrival_time: float
    s_in: int
    s_out: int
    tokens_generated: int = 0


@dataclass(frozen=True)
class ContextInventory:
    """Model shards (layer, lo, hi) and cache shards (rid, layer, lo, hi,
    tokens) one GPU holds (reference: domain.py:175-220)."""

    model_shards: tuple = ()
    cache_shards: tuple = ()

    @staticmethod
    def empty() -> "ContextInventory":
        return ContextInventory()

    def model_intervals(self, layer: int) -> list:
        return [(lo, hi) for lyr, lo, hi in self.model_shards if lyr == layer]

    def cache_entries(self, request_id: str, layer: int) -> list:
        return [((lo, hi), t) for rid, lyr, lo, hi, t in self.cache_shards
                if rid == request_id and lyr == layer]

    def model_bytes(self, model) -> float:
        return float(sum(((hi - lo) * model.bytes_per_layer for _, lo, hi in self.model_shards),
                         Fraction(0)))


@dataclass
class InstanceState:
    """(reference: domain.py:223-248)"""

    id: str
    kind: str
    gpus: int
    status: str = "active"
    grace_deadline: float | None = None
    ready_at: float | None = None
    gpu_inventories: list = field(default_factory=list)

    def __post_init__(self):
        if not self.gpu_inventories:
            self.gpu_inventories = [ContextInventory.empty() for _ in range(self.gpus)]

    def gpu_refs(self) -> list:
        return [(self.id, g) for g in range(self.gpus)]


def stage_layers(num_layers: int, pipeline_stages: int, stage: int) -> range:
    """First L mod P stages take ceil(L/P) layers (reference: domain.py:271-283)."""
    if not 1 <= stage <= pipeline_stages:
        raise DomainError(f"stage {stage} out of 1..{pipeline_stages}")
    q, r = divmod(num_layers, pipeline_stages)
    first = (stage - 1) * q + min(stage - 1, r)
    return range(first, first + q + (1 if stage <= r else 0))


def shard_interval(tensor_shards: int, shard: int) -> Interval:
    """(reference: domain.py:286-288)"""
    return Fraction(shard - 1, tensor_shards), Fraction(shard, tensor_shards)


def required_context(config, pos, model) -> ContextInventory:
    """(reference: domain.py:291-296)"""
    lo, hi = shard_interval(config.tensor_shards, pos.shard)
    block = stage_layers(model.num_layers, config.pipeline_stages, pos.stage)
    return ContextInventory(model_shards=tuple((layer, lo, hi) for layer in block))
