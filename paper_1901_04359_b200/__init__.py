"""B200-native gTop-k S-SGD communication hot path (arXiv 1901.04359).

Drop-in for the reference package `gtopk` (pkg/src/gtopk/__init__.py:3-44):
the same names, argument meanings and exception types, with the compute
running as hand-written sm_100a kernels behind a C ABI (libgtopk_b200.so).

    import paper_1901_04359_b200 as gtopk

Every hot-path name of the reference's top level is exported here.  The
collective and optimizer names are resolved on first use (they import
torch); the reference's TCP mesh (`ClusterConfig`, `connect_tcp_cluster`) is
`tcp.py`, with the collectives staged through host bytes onto this host's
GPU.  The reference's `cost_model` / `models` re-exports are outside this
package's scope.
"""

from .sparse import (
    FLOAT,
    INDEX,
    DeviceSparseVector,
    IndexMask,
    SparseVector,
    as_dense,
    densify,
    k_from_density,
    masked_extract,
    top_k_select,
    top_op,
)
from .transport import (
    DEFAULT_TIMEOUT,
    Endpoint,
    ProtocolError,
    TransportError,
    TransportStats,
    create_local_cluster,
    decode_sparse,
    encode_sparse,
    run_workers,
)
from .tcp import ClusterConfig, TcpEndpoint, connect_tcp_cluster, load_hosts_file

__version__ = "1.1.0"

# reference __init__.py:3-11 (collectives) and :14-24 (optimizer)
_LAZY = {
    "CollectiveStats": "collectives",
    "GTopKResult": "collectives",
    "allgather": "collectives",
    "binomial_bcast": "collectives",
    "dense_ring_allreduce": "collectives",
    "gtopk_allreduce": "collectives",
    "topk_allreduce": "collectives",
    "DensitySchedule": "optimizer",
    "OptimizerState": "optimizer",
    "StepReport": "optimizer",
    "dense_step": "optimizer",
    "density_at": "optimizer",
    "gtopk_naive_step": "optimizer",
    "gtopk_step": "optimizer",
    "make_state": "optimizer",
    "topk_step": "optimizer",
    "STEP_FNS": "optimizer",
    "init_dist_cluster": "dist",
    "GTopKPipeline": "pipeline",
}

__all__ = sorted(
    [
        "FLOAT", "INDEX", "DeviceSparseVector", "IndexMask", "SparseVector", "as_dense", "densify",
        "k_from_density", "masked_extract", "top_k_select", "top_op", "DEFAULT_TIMEOUT", "Endpoint",
        "ProtocolError", "TransportError", "TransportStats", "create_local_cluster", "decode_sparse",
        "encode_sparse", "run_workers", "ClusterConfig", "TcpEndpoint", "connect_tcp_cluster",
        "load_hosts_file",
    ]
    + list(_LAZY)
)


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib

    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(_LAZY))
