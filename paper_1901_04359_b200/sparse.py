"""Dense/sparse gradient vectors, top-k selection and the ⊤ merge -- drop-in
for the reference's `gtopk.sparse` (pkg/src/gtopk/sparse.py).

Host types (`SparseVector`, `IndexMask`) keep the reference's exact data
model (uint64 strictly increasing indices, float32 values).  The compute --
`top_k_select` and `top_op` -- always runs on the GPU through the sm_100a
kernels (K1 select, K2 merge); numpy inputs are copied to the current CUDA
device and results copied back.  torch CUDA inputs stay on the device and
return `DeviceSparseVector` / tensors.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as _dev
from .device import DeviceList

FLOAT = np.float32
INDEX = np.uint64


def as_dense(values) -> np.ndarray:
    """sparse.py:19-24 -- coerce to a 1-D float32 vector."""
    arr = np.asarray(values, dtype=FLOAT)
    if arr.ndim != 1:
        raise ValueError(f"dense vector must be 1-D, got shape {arr.shape}")
    return arr


def k_from_density(rho: float, m: int) -> int:
    """sparse.py:27-31 -- round to nearest (Python banker's rounding), floor 1."""
    if not 0.0 < rho <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {rho}")
    return max(1, min(m, round(rho * m)))


class SparseVector:
    """Host sparse gradient (sparse.py:34-89): dim, uint64 idx, float32 values."""

    __slots__ = ("dim", "indices", "values")

    def __init__(self, dim: int, indices, values):
        self.dim = int(dim)
        self.indices = np.asarray(indices, dtype=INDEX)
        self.values = np.asarray(values, dtype=FLOAT)

    @classmethod
    def empty(cls, dim: int) -> "SparseVector":
        return cls(dim, np.empty(0, dtype=INDEX), np.empty(0, dtype=FLOAT))

    @classmethod
    def from_pairs(cls, dim: int, pairs) -> "SparseVector":
        if not pairs:
            return cls.empty(dim)
        pairs = sorted(pairs)
        return cls(dim, [p[0] for p in pairs], [p[1] for p in pairs])

    @property
    def nnz(self) -> int:
        return len(self.indices)

    def to_pairs(self) -> list[tuple[int, float]]:
        return [(int(i), float(v)) for i, v in zip(self.indices, self.values)]

    def validate(self) -> None:
        if len(self.indices) != len(self.values):
            raise ValueError("index/value length mismatch")
        if len(self.indices) > 0:
            if not np.all(self.indices[:-1] < self.indices[1:]):
                raise ValueError("indices must be strictly increasing")
            if int(self.indices[-1]) >= self.dim:
                raise ValueError("index out of range")

    def to_device(self, device=None, cap=None) -> "DeviceSparseVector":
        dev = device or _dev.default_device()
        return DeviceSparseVector(DeviceList.from_host(self.dim, self.indices, self.values, dev, cap))

    def __eq__(self, other) -> bool:
        if isinstance(other, DeviceSparseVector):
            other = other.to_host()
        if not isinstance(other, SparseVector):
            return NotImplemented
        return (
            self.dim == other.dim
            and np.array_equal(self.indices, other.indices)
            and np.array_equal(self.values, other.values)
        )

    __hash__ = None

    def __repr__(self) -> str:
        return f"SparseVector(dim={self.dim}, entries={self.to_pairs()})"


class DeviceSparseVector:
    """A sparse vector resident in HBM (int32 idx / f32 val / device count)."""

    __slots__ = ("list",)

    def __init__(self, lst: DeviceList):
        self.list = lst

    @property
    def dim(self) -> int:
        return self.list.dim

    @property
    def nnz(self) -> int:
        return self.list.nnz()

    def to_host(self) -> SparseVector:
        i, v = self.list.to_host()
        return SparseVector(self.list.dim, i, v)

    @property
    def indices(self) -> np.ndarray:
        return self.to_host().indices

    @property
    def values(self) -> np.ndarray:
        return self.to_host().values

    def to_pairs(self):
        return self.to_host().to_pairs()

    def __eq__(self, other) -> bool:
        return self.to_host() == other

    __hash__ = None

    def __repr__(self) -> str:
        return f"DeviceSparseVector(dim={self.dim}, nnz={self.nnz}, device={self.list.device})"


class IndexMask:
    """{0,1} selection over a dense dimension (sparse.py:92-132).

    Masks built from a sorted index list (the global top-k set) stay lazy:
    the m-byte flag array is only materialised on `.flags` access.
    """

    def __init__(self, dim: int, flags=None, *, _indices=None):
        self.dim = int(dim)
        self._indices = None
        self._flags = None
        if _indices is not None:
            self._indices = np.asarray(_indices, dtype=INDEX)
        else:
            f = np.asarray(flags, dtype=bool)
            if f.shape != (self.dim,):
                raise ValueError("mask flags must have shape (dim,)")
            self._flags = f

    @classmethod
    def from_indices(cls, dim: int, indices) -> "IndexMask":
        idx = np.asarray(indices, dtype=INDEX)
        if len(idx) and int(idx.max()) >= dim:
            raise ValueError("mask index out of range")
        idx = np.unique(idx)
        return cls(dim, _indices=idx)

    @property
    def flags(self) -> np.ndarray:
        if self._flags is None:
            f = np.zeros(self.dim, dtype=bool)
            f[self._indices] = True
            self._flags = f
        return self._flags

    @flags.setter
    def flags(self, value) -> None:
        f = np.asarray(value, dtype=bool)
        if f.shape != (self.dim,):
            raise ValueError("mask flags must have shape (dim,)")
        self._flags = f
        self._indices = None

    @property
    def indices(self) -> np.ndarray:
        if self._indices is not None and self._flags is None:
            return self._indices.copy()
        return np.nonzero(self.flags)[0].astype(INDEX)

    @property
    def count(self) -> int:
        if self._indices is not None and self._flags is None:
            return int(self._indices.size)
        return int(self.flags.sum())

    def __invert__(self) -> "IndexMask":
        return IndexMask(self.dim, ~self.flags)

    def __and__(self, other: "IndexMask") -> "IndexMask":
        if self.dim != other.dim:
            raise ValueError("mask dimension mismatch")
        return IndexMask(self.dim, self.flags & other.flags)

    def __eq__(self, other) -> bool:
        if not isinstance(other, IndexMask):
            return NotImplemented
        return self.dim == other.dim and np.array_equal(self.indices, other.indices)

    __hash__ = None


# ---------------------------------------------------------------------------
# compute entry points (GPU)
# ---------------------------------------------------------------------------


def _is_cuda_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def top_k_select(g, k: int):
    """sparse.py:135-154 on the GPU (kernel K1).

    numpy/list in  -> (SparseVector, np.ndarray residual)
    CUDA tensor in -> (DeviceSparseVector, residual tensor)
    Exactly k entries, ties toward the lower index, values copied bitwise, the
    residual zeroed (+0.0) at the kept slots; FloatingPointError on NaN/Inf.
    """
    on_device = _is_cuda_tensor(g)
    if on_device:
        if g.dim() != 1:
            raise ValueError(f"dense vector must be 1-D, got shape {tuple(g.shape)}")
        gd = g.contiguous().to(torch.float32)
        dev = gd.device
        m = gd.numel()
    else:
        gh = as_dense(g)
        m = gh.size
    if not 1 <= k <= m:
        raise ValueError(f"k must be in [1, {m}], got {k}")
    if not on_device:
        dev = _dev.default_device()
        gd = torch.from_numpy(np.ascontiguousarray(gh)).to(dev)
    res = torch.empty_like(gd)
    out = DeviceList(m, k, dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _dev.select(None, gd, res, k, out, status)
    word = int(status.item())
    _dev.raise_status(word)
    if on_device:
        return DeviceSparseVector(out), res
    i, v = out.to_host()
    return SparseVector(m, i, v), res.cpu().numpy()


def _as_device_list(s, device, cap):
    if isinstance(s, DeviceSparseVector):
        return s.list
    return DeviceList.from_host(s.dim, s.indices, s.values, device, cap)


def top_op(a, b, k: int):
    """sparse.py:157-195 on the GPU (kernel K2): a+b on shared indices, exact
    zeros dropped, the k largest |v| kept (ties -> lower index), index order.

    Host SparseVectors in -> SparseVector out; any DeviceSparseVector in ->
    DeviceSparseVector out."""
    if a.dim != b.dim:
        raise ValueError(f"dimension mismatch: {a.dim} != {b.dim}")
    if k < 1:
        raise ValueError(f"k must be positive, got {k}")
    on_device = isinstance(a, DeviceSparseVector) or isinstance(b, DeviceSparseVector)
    if on_device:
        dev = (a if isinstance(a, DeviceSparseVector) else b).list.device
    else:
        if a.nnz == 0 and b.nnz == 0:
            return SparseVector.empty(a.dim)
        dev = _dev.default_device()
    na_cap = a.list.cap if isinstance(a, DeviceSparseVector) else max(a.nnz, 1)
    nb_cap = b.list.cap if isinstance(b, DeviceSparseVector) else max(b.nnz, 1)
    cap = max(na_cap, nb_cap)
    la = _as_device_list(a, dev, cap)
    lb = _as_device_list(b, dev, cap)
    out = DeviceList(a.dim, max(min(k, la.cap + lb.cap), 1), dev)
    _dev.top_op(la, lb, k, out)
    if on_device:
        return DeviceSparseVector(out)
    i, v = out.to_host()
    return SparseVector(a.dim, i, v)


def densify(s) -> np.ndarray:
    """sparse.py:198-202 -- zero-filled dense vector with s's entries.

    DeviceSparseVector -> CUDA tensor (kernel); SparseVector -> numpy."""
    if isinstance(s, DeviceSparseVector):
        out = torch.empty(s.dim, dtype=torch.float32, device=s.list.device)
        _dev.densify(s.list, s.dim, out)
        return out
    out = np.zeros(s.dim, dtype=FLOAT)
    out[s.indices] = s.values
    return out


def masked_extract(g, keep: IndexMask) -> np.ndarray:
    """sparse.py:205-210 -- values of g where the mask is set, zero elsewhere."""
    g = as_dense(g)
    if g.size != keep.dim:
        raise ValueError(f"dimension mismatch: {g.size} != {keep.dim}")
    return np.where(keep.flags, g, FLOAT(0))
