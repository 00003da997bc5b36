"""B200-native sparse MPM: the hash-grid time step of "Unified sparse
framework for large-scale MPM" (arxiv/paper_2605_28525) on sm_100a.

Drop-in for the reference package ``sparsempm``'s hash path
(/root/reference/pkg/src/sparsempm/): same classes and functions, computed by
hand-written CUDA kernels in ``libsmpm.so`` (C ABI: include/smpm.h).
"""

from .errors import ConfigError, InactiveNodeError, KeyRangeError, SimulationError, SparseMpmError
from .grid_index import ActiveIndexMap, block_of, local_offset, mix64, node_index, pack_key, unpack_key
from .materials import MaterialModel, update_stress
from .solver import (
    BoundaryCondition,
    Heightfield,
    NodalFields,
    ParticleSet,
    SimConfig,
    Simulation,
    StepStats,
    apply_friction_boundary,
    bspline_weights,
    count_active_nodes,
    g2p,
    grid_forces,
    grid_update,
    p2g,
)
from .sparse_hash import BlockHashTable, build_hash_sparse_grid
from .scenarios import load_config, load_heightfield, sample_box
from .bench import compare, run, sliding_box_oracle, sparsity_ratio

__version__ = "0.1.0"

__all__ = [
    "ActiveIndexMap", "BlockHashTable", "BoundaryCondition", "ConfigError", "Heightfield", "InactiveNodeError",
    "KeyRangeError", "MaterialModel", "NodalFields", "ParticleSet", "SimConfig", "Simulation", "SimulationError",
    "SparseMpmError", "StepStats", "apply_friction_boundary", "block_of", "bspline_weights",
    "build_hash_sparse_grid", "count_active_nodes", "g2p", "grid_forces", "grid_update", "local_offset", "mix64",
    "node_index", "p2g", "pack_key", "unpack_key", "update_stress", "load_config", "load_heightfield", "sample_box",
    "compare", "run", "sliding_box_oracle", "sparsity_ratio",
]
