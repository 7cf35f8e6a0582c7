"""B200-native top-down BFS (arXiv 1604.02844's path), a drop-in for the
reference package ``lanebfs`` on its hot path.

Graph inputs (graph.py), the device BFS (traversal.py -> liblbfs.so, sm_100a),
the tree validator (validate.py) and the TEPS harness (harness.py) keep the
reference names and result types (/root/reference/pkg/src/lanebfs/__init__.py).
"""

from .graph import (
    MAX_SCALE,
    CsrGraph,
    EdgeList,
    RmatParams,
    build_csr,
    build_lattice_graph,
    build_rmat_graph,
    generate_rmat,
    lattice_edges,
    permutation_seed,
    permute_vertices,
    read_edge_list,
    write_edge_list,
)
from .harness import (
    ExperimentConfig,
    RootRun,
    RunStats,
    emit_results,
    harmonic_mean_teps,
    pick_roots,
    run_experiment,
)
from .traversal import (
    MODES,
    SENTINEL,
    BfsResult,
    LayerPolicy,
    LayerStats,
    PredecessorArray,
    bfs,
    bfs_device,
    run_bfs,
)
from .validate import (
    Certificate,
    ValidationReport,
    bfs_certificate,
    levels_from_parents,
    validate_tree,
    validate_tree_device,
)

__all__ = [
    "MAX_SCALE", "CsrGraph", "EdgeList", "RmatParams", "build_csr", "build_lattice_graph",
    "build_rmat_graph", "generate_rmat", "lattice_edges", "permutation_seed", "permute_vertices",
    "read_edge_list", "write_edge_list", "ExperimentConfig", "RootRun", "RunStats", "emit_results",
    "harmonic_mean_teps", "pick_roots", "run_experiment", "MODES", "SENTINEL", "BfsResult",
    "LayerPolicy", "LayerStats", "PredecessorArray", "bfs", "bfs_device", "run_bfs", "Certificate",
    "ValidationReport", "bfs_certificate", "levels_from_parents", "validate_tree", "validate_tree_device",
]

__version__ = "0.1.0"
