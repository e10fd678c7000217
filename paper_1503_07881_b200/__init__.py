"""B200-native drop-in for the graphtables hot path (ToGraph, PageRank, triangles).

The import surface mirrors the reference package ``graphtables``
(``pkg/src/graphtables/__init__.py``) for everything on the path:
``ColumnTable``, ``Schema``, ``EdgeSpec``, ``table_to_graph``, ``pagerank``,
``triangle_count``, ``Graph``, ``NodeRecord``, ``from_edges``, ``load_tsv`` and
the error types. Compute runs only in ``libgtb200.so`` (hand-written sm_100a
CUDA, C ABI in ``include/gtb200.h``); importing this package never touches
the GPU, calling the path without the library raises ``NativeError``.
"""

from .algorithms import (DistMap, LabelMap, RankMap, connected_components, k_core, pagerank,
                         pagerank_and_triangles, pagerank_device, scc, sssp,
                         triangle_count)
from .convert import EdgeSpec, graph_to_edge_table, graph_to_node_table, table_to_graph
from .errors import (
    CapacityError,
    CoverageError,
    EngineError,
    NativeError,
    ParseError,
    SchemaError,
    TypeMismatchError,
    UnknownColumnError,
    UnknownNodeError,
)
from .graph import DeviceGraph, Graph, NodeRecord, from_edges, upload
from .relational import Predicate, join, project, select
from .tables import (FLOAT, INT, STRING, ColumnTable, Schema, edge_table, load_tsv, save_tsv,
                     table_from_map)

__version__ = "0.1.0"

__all__ = [
    "CapacityError", "ColumnTable", "CoverageError", "DeviceGraph", "EdgeSpec", "EngineError",
    "FLOAT", "Graph", "INT", "NativeError", "NodeRecord", "ParseError", "RankMap", "STRING",
    "Schema", "SchemaError", "TypeMismatchError", "UnknownColumnError", "UnknownNodeError",
    "edge_table", "from_edges", "graph_to_edge_table", "graph_to_node_table", "load_tsv",
    "pagerank", "pagerank_device", "save_tsv", "table_from_map", "table_to_graph",
    "triangle_count", "upload", "sssp", "connected_components", "k_core", "DistMap",
    "LabelMap", "scc", "pagerank_and_triangles", "Predicate", "select", "project", "join",
]
