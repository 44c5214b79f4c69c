"""B200-native edge-centric graphlet census (arXiv 1506.04322).

Drop-in for the counting entry points of the reference package ``graphlets``
(graphlets/__init__.py:10-56): same names, signatures, result types and
error classes, with the per-edge counting, the schedule and the reductions
running as hand-written sm_100a kernels in libgdgpu.so (C ABI:
include/gd_api.h).  There is no CPU fallback.
"""

from .analytics import (RANK_PATTERNS, FeatureMatrix, GfdVector, RankedEdge, edge_weights,
                        feature_matrix, gfd, rank_edges, vertex_triangle_counts)
from .census import (RAW_MICRO_FIELDS, CensusSums, census_batch, close_quads,
                     close_triads, frequencies_from_micro, frequencies_from_sums,
                     graphlet_census, last_stats, last_timings, micro_census_table,
                     micro_table, trim_workspace)
from .edgelist import load_edge_list, to_edge_list_text
from .classes import (ALL_CLASSES, CLASS_BY_ID, CLASS_IDS, GraphletClass,
                      classes_for, complement_class)
from .errors import (ClassificationError, ConsistencyError, DeviceError,
                     EdgeListParseError, GraphletError, GraphSizeError)
from .frequencies import GraphletFrequencies
from .graph import EdgeRef, Graph, GraphBatch, ParseOptions, order_edges_by_degree
from .introspect import (clear_marks, clique_count, cycle_count, edge_neighborhood_census,
                         same_side_star_edges)
from .micro import (MICRO_CSV_HEADER, EdgeLocalCounts, MicroCounts, UnrestrictedCounts,
                    derive_micro, micro_census, micro_counts_from_table, micro_csv,
                    micro_roles, write_micro_csv, ROLE_COLUMNS,
                    unrestricted_counts)
from .parallel import MAX_BATCH_SIZE, ParallelConfig, WorkerFailure
from .selection import SelectionOp, SelectionState, induced_subgraph, selection_census

__version__ = "0.1.0"

__all__ = [
    "FeatureMatrix", "GfdVector", "feature_matrix", "gfd",
    "RANK_PATTERNS", "RankedEdge", "edge_weights", "rank_edges", "vertex_triangle_counts",
    "RAW_MICRO_FIELDS", "CensusSums", "census_batch", "close_quads", "close_triads",
    "frequencies_from_micro", "frequencies_from_sums", "graphlet_census", "last_stats",
    "last_timings", "micro_census_table", "micro_table", "trim_workspace",
    "ALL_CLASSES", "CLASS_BY_ID", "CLASS_IDS", "GraphletClass", "classes_for",
    "complement_class",
    "ClassificationError", "ConsistencyError", "DeviceError", "EdgeListParseError",
    "GraphletError", "GraphSizeError",
    "GraphletFrequencies",
    "EdgeRef", "Graph", "GraphBatch", "ParseOptions", "order_edges_by_degree",
    "load_edge_list", "to_edge_list_text",
    "MAX_BATCH_SIZE", "ParallelConfig", "WorkerFailure",
    "SelectionOp", "SelectionState", "induced_subgraph", "selection_census",
    "MICRO_CSV_HEADER", "EdgeLocalCounts", "MicroCounts", "UnrestrictedCounts", "derive_micro",
    "micro_census", "micro_counts_from_table", "micro_csv", "unrestricted_counts",
    "micro_roles", "write_micro_csv", "ROLE_COLUMNS",
    "clear_marks", "clique_count", "cycle_count", "edge_neighborhood_census",
    "same_side_star_edges",
    "__version__",
]
