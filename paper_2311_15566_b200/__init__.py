"""B200-native SpotServe (arXiv 2311.15566) device-mapping + context-migration path.

Drop-in for the reference package's mapper/planner API (`spotsim`,
reference __init__.py:61-79): the same function names, arguments, results and
exceptions, computed by hand-written sm_100a kernels behind a C ABI
(include/spotkm.h, libspotkm.so).  `install(spotsim)` rebinds the reference's
names to these implementations.
"""

__version__ = "0.1.0"

from .domain import (  # noqa: F401
    ContextInventory,
    InstanceState,
    ModelSpec,
    ParallelConfig,
    RequestSpec,
    TopologyPosition,
    positions,
    required_context,
)
from .mapping import (  # noqa: F401
    BipartiteGraph,
    DeviceMapping,
    MappingError,
    build_graph,
    default_inheritance,
    km_match,
    map_devices,
    map_devices_many,
)
from .migration import MigrationAction, MigrationError, MigrationPlan, Transfer  # noqa: F401
from .planner import (  # noqa: F401
    LayerTraffic,
    derive_transfers,
    memopt_layer_order,
    migration_cost,
    plan_from_dict,
    plan_migration,
    plan_migration_many,
    plan_timeline,
    plan_to_dict,
    simulate_buffer_usage,
)
from .estimator import (  # noqa: F401
    exec_latency_many,
    optimize_config_many,
    throughput_many,
)
