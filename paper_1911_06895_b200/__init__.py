"""B200-native drop-in for the reference's delta-stepping SSSP path.

Public names follow the reference package `deltasparse` for this path
(/root/reference/pkg/src/deltasparse/__init__.py): `delta_stepping`,
`SsspResult`, `split_edges`, `BackendChoice`, `bucket_bounds`, the
`SparseMatrix` / `SparseVector` containers and their builders, and the graph
file loaders (`load_matrix_market`, `load_edge_list`, `load_graph`, parsed
natively).  Compute runs
in libdsssp.so (sm_100a) through the C-ABI declared in include/dsssp.h.
"""

from .containers import (  # noqa: F401
    SparseMatrix,
    SparseVector,
    mask_from_indices,
    matrix_build,
    vector_build,
)
from .io import (  # noqa: F401
    GraphFile,
    GraphLoadError,
    LabelMap,
    ParseError,
    ValidationError,
    load_edge_list,
    load_graph,
    load_csr,
    load_matrix_market,
    save_csr,
)
from .sssp import (  # noqa: F401
    BackendChoice,
    DeviceGraph,
    SsspResult,
    bucket_bounds,
    clear_device_cache,
    clear_host_buffers,
    delta_stepping,
    delta_stepping_batch,
    split_edges,
)

__version__ = "0.1.0"

__all__ = [
    "SparseMatrix",
    "SparseVector",
    "mask_from_indices",
    "matrix_build",
    "vector_build",
    "BackendChoice",
    "DeviceGraph",
    "SsspResult",
    "bucket_bounds",
    "clear_device_cache",
    "clear_host_buffers",
    "delta_stepping",
    "delta_stepping_batch",
    "split_edges",
    "GraphFile",
    "GraphLoadError",
    "LabelMap",
    "ParseError",
    "ValidationError",
    "load_edge_list",
    "load_graph",
    "load_matrix_market",
    "load_csr",
    "save_csr",
    "__version__",
]
