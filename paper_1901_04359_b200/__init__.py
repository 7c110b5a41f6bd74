"""B200-native gTop-k S-SGD communication hot path (arXiv 1901.04359).

Drop-in for the reference package `gtopk` (pkg/src/gtopk/__init__.py:3-44):
the same names, argument meanings and exception types, with the compute
running as hand-written sm_100a kernels behind a C ABI (libgtopk_b200.so).

    import paper_1901_04359_b200 as gtopk
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

__version__ = "1.0.0"
