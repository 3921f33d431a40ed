"""Rebind the reference package's hot-path names to this implementation.

The reference's simulator binds `map_devices`, `plan_migration`,
`derive_transfers` and `migration_cost` by name at import
(simulator.py:30-61), and user code imports them from `spotsim`,
`spotsim.mapping`, `spotsim.migration` and `spotsim.costmodel`
(__init__.py:33-79).  `install(spotsim)` replaces every such binding so that
existing callers run on the B200 path unchanged; `uninstall()` restores them.

    import spotsim
    from paper_2311_15566_b200.install import install
    install(spotsim)                       # everything
    install(spotsim, parts=("planner",))   # only the native planner/estimator
"""

from __future__ import annotations

import sys

from . import estimator as _estimator
from . import mapping as _mapping
from . import planner as _planner

PARTS = {
    "mapper": {"build_graph": _mapping.build_graph, "km_match": _mapping.km_match,
               "map_devices": _mapping.map_devices},
    "planner": {"plan_migration": _planner.plan_migration,
                "derive_transfers": _planner.derive_transfers,
                "memopt_layer_order": _planner.memopt_layer_order,
                "simulate_buffer_usage": _planner.simulate_buffer_usage},
    "estimator": {"plan_timeline": _planner.plan_timeline,
                  "migration_cost": _planner.migration_cost},
    # opt-in: device-batched candidate scoring; per single call it pays a
    # device round trip, so the default install leaves the reference's here
    "controller": {"exec_latency": _estimator.exec_latency, "throughput": _estimator.throughput,
                   "optimize_config": _estimator.optimize_config},
}

_saved: list = []


def install(pkg, parts=("mapper", "planner", "estimator")) -> list:
    """Rebind names in `pkg` and its already-imported submodules.  Returns the
    list of (module, name) pairs replaced."""
    names = {}
    for part in parts:
        names.update(PARTS[part])
    prefix = pkg.__name__
    mods = [m for k, m in sorted(sys.modules.items()) if m is not None
            and (k == prefix or k.startswith(prefix + "."))]
    done = []
    for mod in mods:
        for name, fn in names.items():
            if name in vars(mod):
                _saved.append((mod, name, vars(mod)[name]))
                setattr(mod, name, fn)
                done.append((mod.__name__, name))
    return done


def uninstall() -> None:
    while _saved:
        mod, name, old = _saved.pop()
        setattr(mod, name, old)
