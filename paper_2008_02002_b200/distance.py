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


def packed_distance(x: PackedVector, y: PackedVector) -> int:
    """distance.py:32-41: pairwise XOR/popcount distance; widths may differ, dims must match.  One-row use of the
    distance kernel (the definition twin of batch_distances)."""
    if x.dim != y.dim:
        raise DimensionMismatchError(f"dim mismatch: {x.dim} vs {y.dim}")
    if x.dim == 0:
        return 0
    return int(batch_distances(PackedMatrix(np.ascontiguousarray(x.planes[:, :, None]), x.dim), y)[0])


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
    with torch.cuda.device(matrix.device):
        q = query.device_words(matrix.device)
        d = torch.empty(matrix.count, dtype=torch.int64, device=matrix.device)
        _native.check(L.xfbq_batch_distances(matrix.codes.data_ptr(), matrix.count, matrix.dim, matrix.width,
                                             q.data_ptr(), query.width, d.data_ptr(), _stream_ptr(torch)))
    return d


def collect_candidates_device(matrix: PackedMatrix, query, threshold: int, want_ids: bool, cap: int = 1 << 16, query_bits: int | None = None):
    """Number of rows with distance <= threshold and (want_ids) their row ids as a device int64 tensor, unordered:
    the histogram/gather stage of k_select (search.py:206-216) in one pass over the codes, without the distance
    array.  `query`: a PackedVector, or device query words (query layout, with `query_bits`).  The pass runs on the nibble
    layout when the index has built it (dp4a, HBM-bound), else on the bit planes (XOR/POPC).  The id buffer grows to the
    count when `cap` was too small (second pass)."""
    torch = _native.require_cuda()
    L = _native.lib()
    dev = matrix.device
    with torch.cuda.device(dev):
        if isinstance(query, PackedVector):
            q, wq = query.device_words(dev), query.width
        else:
            q, wq = query, int(query_bits)
        nib = getattr(matrix, "_nibbles", None) if wq <= 7 else None
        count_dev = torch.empty(1, dtype=torch.int64, device=dev)
        while True:
            ids = torch.empty(cap if want_ids else 0, dtype=torch.int64, device=dev)
            if nib is not None:
                _native.check(L.xfbq_collect_candidates_nibbles(nib.data_ptr(), matrix.count, matrix.dim, matrix.width, q.data_ptr(), wq,
                                                                int(threshold), ids.data_ptr() if want_ids else None, cap,
                                                                count_dev.data_ptr(), _stream_ptr(torch)))
            else:
                _native.check(L.xfbq_collect_candidates(matrix.codes.data_ptr(), matrix.count, matrix.dim, matrix.width,
                                                        q.data_ptr(), wq, int(threshold),
                                                        ids.data_ptr() if want_ids else None, cap, count_dev.data_ptr(), _stream_ptr(torch)))
            count = int(count_dev.item())
            if not want_ids or count <= cap:
                return count, (ids[:count] if want_ids else None)
            cap = count


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
