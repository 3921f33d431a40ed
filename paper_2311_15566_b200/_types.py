"""Resolve the caller's result classes.

The reference's tests compare results with `==` on dataclasses, which only
holds between instances of the SAME class (e.g. `fused.assignment ==
flat.assignment`, tests/test_mapping.py:209).  So results are built with the
classes of the package the caller's inputs come from: when the inputs are
`spotsim` objects the results are `spotsim.mapping.DeviceMapping` /
`spotsim.domain.TopologyPosition` etc.; otherwise this package's own.
"""

from __future__ import annotations

import sys
from types import SimpleNamespace


def _own():
    from . import domain, mapping, migration

    return SimpleNamespace(
        TopologyPosition=domain.TopologyPosition,
        ContextInventory=domain.ContextInventory,
        BipartiteGraph=mapping.BipartiteGraph,
        DeviceMapping=mapping.DeviceMapping,
        MappingError=mapping.MappingError,
        Transfer=migration.Transfer,
        MigrationAction=migration.MigrationAction,
        MigrationPlan=migration.MigrationPlan,
        MigrationError=migration.MigrationError,
    )


_cache: dict[str, SimpleNamespace] = {}


def result_types(obj) -> SimpleNamespace:
    """Classes of the package `obj`'s type lives in (falls back to ours)."""
    mod = type(obj).__module__ or ""
    pkg = mod.rsplit(".", 1)[0] if "." in mod else mod
    if pkg in _cache:
        return _cache[pkg]
    own = _own()
    if pkg == __package__:
        _cache[pkg] = own
        return own
    dom = sys.modules.get(f"{pkg}.domain")
    mp = sys.modules.get(f"{pkg}.mapping")
    mg = sys.modules.get(f"{pkg}.migration")
    ns = SimpleNamespace(**vars(own))
    if dom is not None:
        for name in ("TopologyPosition", "ContextInventory"):
            if hasattr(dom, name):
                setattr(ns, name, getattr(dom, name))
    if mp is not None:
        for name in ("BipartiteGraph", "DeviceMapping", "MappingError"):
            if hasattr(mp, name):
                setattr(ns, name, getattr(mp, name))
    if mg is not None:
        for name in ("Transfer", "MigrationAction", "MigrationPlan", "MigrationError"):
            if hasattr(mg, name):
                setattr(ns, name, getattr(mg, name))
    _cache[pkg] = ns
    return ns
