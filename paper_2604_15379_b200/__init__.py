"""B200-native hierarchical task megakernel for Qwen3 decode.

Drop-in for the task-graph API of the reference package ``chipletsim``
(``/root/reference/pkg/src/chipletsim/__init__.py:13-73``): the same names
build the same graphs.  Instead of the reference's CPU simulation
(``simulate``), :mod:`.runtime` lowers a graph to device descriptors and runs
one decode step per launch of a persistent sm_100a kernel through the C-ABI
declared in ``include/mk.h``.
"""

from .machine import (ConfigError, MachineConfig, ModelConfig, b200_from_probe,
                      load_machine, load_model, model_preset, preset,
                      resolve_machine, resolve_model, validate, validate_model)
from .taskgraph import (LINEAR_OPS, STANDARD_TILE_PROFILE, ElementwiseWork,
                        Event, GemmTileWork, GemmWork, GraphError, OpaqueWork,
                        OpKind, StageRecord, Task, TaskGraph, TaskLevel,
                        build_decoder_layer, build_gemm_graph,
                        cross_chiplet_event_reduction, graph_to_dot,
                        graph_to_json, validate_graph, worker_multiplicity)
from .traversal import (Distribution, GemmPartition, ScheduleError,
                        TileSchedule, Traversal, schedule, schedule_to_json)

__version__ = "0.1.0"

# reference mode names -> (graph mode, traversal, distribution)
# (ref scenario.py:37-46)
MODES = {
    "standard": ("standard", Traversal.M_MAJOR_WINDOWED, Distribution.M_TILE),
    "chiplet_m_tile": ("chiplet", Traversal.M_MAJOR_WINDOWED,
                       Distribution.M_TILE),
    "chiplet_m_split": ("chiplet", Traversal.M_MAJOR_WINDOWED,
                        Distribution.M_SPLIT),
    "chiplet_n_major": ("chiplet", Traversal.N_MAJOR, Distribution.M_TILE),
}
