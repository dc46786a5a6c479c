"""batch_distances / distance_upper_bound / decode (reference distance.py:25-83)."""
from __future__ import annotations

import numpy as np

from . import _native
from .bitplane import PackedMatrix, PackedVector, _stream_ptr, check_width
from .errors import DimensionMismatchError, InvalidInputError


def scalar_product_upper_bound(width_x: int, width_y: int) -> int:
    """quant.py:113-115."""
    return ((1 << check_width(width_x)) - 1) * ((1 << check_width(width_y)) - 1)


def distance_upper_bound(dim: int, width_x: int, width_y: int) -> int:
    """distance.py:25-29."""
    if dim < 0:
        raise InvalidInputError(f"dim must be non-negative, got {dim}")
    return int(dim) * scalar_product_upper_bound(width_x, width_y)


def batch_distances(matrix: PackedMatrix, query: PackedVector, out: np.ndarray | None = None) -> np.ndarray:
    """distance.py:44-62: uint64[n] distances from one packed query to every row, computed by
    the CUDA distance kernel and copied to the host (or into the caller's `out`)."""
    if matrix.dim != query.dim:
        raise DimensionMismatchError(f"dim mismatch: {matrix.dim} vs {query.dim}")
    n = matrix.count
    if out is None:
        out = np.empty(n, dtype=np.uint64)
    elif out.shape != (n,) or out.dtype != np.uint64:
        raise InvalidInputError("out buffer must be uint64 of length matrix.count")
    if n == 0:
        return out
    dev = batch_distances_device(matrix, query)
    out[:] = dev.cpu().numpy().view(np.uint64)
    return out


def batch_distances_device(matrix: PackedMatrix, query: PackedVector):
    """Device-resident int64[n] distances (same values)."""
    torch = _native.require_cuda()
    L = _native.lib()
    with torch.cuda.device(matrix.codes.device):
        q = query.device_words()
        d = torch.empty(matrix.count, dtype=torch.int64, device=matrix.codes.device)
        _native.check(L.xfbq_batch_distances(matrix.codes.data_ptr(), matrix.count, matrix.dim, matrix.width,
                                             q.data_ptr(), query.width, d.data_ptr(), _stream_ptr(torch)))
    return d


def decode_inner_product(d: int, dim: int, width_x: int, width_y: int) -> float:
    """distance.py:65-74."""
    hi = distance_upper_bound(dim, width_x, width_y)
    if not 0 <= int(d) <= hi:
        raise InvalidInputError(f"distance {d} outside [0, {hi}]")
    return (hi - 2 * int(d)) / float(1 << (width_x + width_y))


def decode_inner_product_values(d, dim: int, width_x: int, width_y: int) -> np.ndarray:
    """distance.py:77-83: (hi - 2d) / 2^(wx+wy) in float64, exact (dyadic)."""
    hi = float(distance_upper_bound(dim, width_x, width_y))
    return (hi - 2.0 * np.asarray(d, dtype=np.float64)) / float(1 << (width_x + width_y))
