"""Packed bit-plane containers and the GPU quantizer front end.

Mirrors the reference's `bitplane.py` surface (/root/reference/pkg/src/xfbq/bitplane.py):
`PackedVector`, `PackedMatrix`, `quantize_vector`, `quantize_matrix`, `pack_matrix`,
`unpack_matrix`, `words_needed`.  A `PackedMatrix` here owns the codes in HBM in the
bundle layout (include/xfbq_b200.h); the reference's word-major `(width, words, n)`
uint64 array is available through `.planes` (converted on the GPU, copied to the host on
first use, read-only like the reference's, bitplane.py:98).
"""
from __future__ import annotations

import numpy as np

from . import _native
from .errors import InvalidInputError

WORD_BITS = 64
MAX_WIDTH = 8
_ROW_CHUNK = 1 << 20  # rows staged per host->device copy when quantizing host matrices


def check_width(width) -> int:
    """quant.py:23-31."""
    w = int(width)
    if w < 1 or w > MAX_WIDTH:
        raise InvalidInputError(f"bit width must be in 1..{MAX_WIDTH}, got {width}")
    return w


def words_needed(dim: int) -> int:
    """bitplane.py:29-30."""
    return (int(dim) + WORD_BITS - 1) // WORD_BITS


def _padding_ok(planes: np.ndarray, dim: int) -> bool:
    """bitplane.py:33-46: bits past `dim` in the last word must be zero."""
    if dim == 0 or planes.size == 0 or dim % WORD_BITS == 0:
        return True
    mask = np.uint64((1 << (dim % WORD_BITS)) - 1)
    last = planes[:, -1] if planes.ndim == 2 else planes[:, -1, :]
    return not np.any(last & ~mask)


def _stream_ptr(torch):
    return torch.cuda.current_stream().cuda_stream


class PackedVector:
    """One quantized vector as ``(width, words)`` uint64 bit-planes (bitplane.py:49-76)."""

    __slots__ = ("planes", "dim")

    def __init__(self, planes, dim: int):
        planes = np.ascontiguousarray(planes, dtype=np.uint64)
        if planes.ndim != 2:
            raise InvalidInputError("planes must be a (width, words) array")
        check_width(planes.shape[0])
        if dim < 0 or planes.shape[1] != words_needed(dim):
            raise InvalidInputError(
                f"expected {words_needed(dim)} words per plane for dim {dim}, got {planes.shape[1]}")
        if not _padding_ok(planes, dim):
            raise InvalidInputError("nonzero padding bits past the true dimension")
        planes.setflags(write=False)
        object.__setattr__(self, "planes", planes)
        object.__setattr__(self, "dim", int(dim))

    def __setattr__(self, key, value):  # frozen, like the reference dataclass
        raise AttributeError("PackedVector is immutable")

    @property
    def width(self) -> int:
        return self.planes.shape[0]

    @property
    def nbytes(self) -> int:
        return self.planes.nbytes

    def device_words(self, device=None):
        """Query layout uint32 [1][width][4C] on `device` (default: the current CUDA device)."""
        torch = _native.require_cuda()
        C = (self.dim + 127) // 128
        host = np.zeros((self.width, 2 * C), dtype=np.uint64)
        host[:, : self.planes.shape[1]] = self.planes
        return torch.from_numpy(host.view(np.int64).reshape(1, -1)).to(device if device is not None else "cuda")


class PackedMatrix:
    """n quantized vectors; codes live in HBM in the bundle layout.

    Reference surface (bitplane.py:79-122): ``planes`` (word-major ``(width, words, n)``
    uint64, read-only), ``dim``, ``width``, ``count``, ``nbytes``, ``row(k)``,
    ``to_row_major()``, ``from_row_major()``.
    """

    def __init__(self, planes=None, dim: int | None = None, *, _codes=None, _count=None, _width=None):
        if dim is None:
            raise InvalidInputError("dim is required")
        self._dim = int(dim)
        self._planes = None
        if _codes is not None:  # device path (quantizer output)
            self._codes, self._count, self._width = _codes, int(_count), int(_width)
            return
        planes = np.ascontiguousarray(planes, dtype=np.uint64)
        if planes.ndim != 3:
            raise InvalidInputError("planes must be a (width, words, n) array")
        check_width(planes.shape[0])
        if self._dim < 0 or planes.shape[1] != words_needed(self._dim):
            raise InvalidInputError(
                f"expected {words_needed(self._dim)} words per plane for dim {self._dim}, got {planes.shape[1]}")
        if not _padding_ok(planes, self._dim):
            raise InvalidInputError("nonzero padding bits past the true dimension")
        if self._dim < 1:
            raise InvalidInputError("dim must be >= 1 for a device-resident matrix")
        planes.setflags(write=False)
        self._planes = planes
        self._width, self._count = planes.shape[0], planes.shape[2]
        torch = _native.require_cuda()
        L = _native.lib()
        self._codes = torch.empty(max(int(L.xfbq_db_bytes(self._count, self._dim, self._width)), 16),
                                  dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
        if self._count:
            dev = torch.from_numpy(planes.view(np.int64)).to(self._codes.device)
            _native.check(L.xfbq_planes_to_bundles(dev.data_ptr(), self._count, self._dim, self._width,
                                                   self._codes.data_ptr(), _stream_ptr(torch)))
            torch.cuda.current_stream().synchronize()

    # ---- reference surface
    @property
    def dim(self) -> int:
        return self._dim

    @property
    def width(self) -> int:
        return self._width

    @property
    def count(self) -> int:
        return self._count

    @property
    def nbytes(self) -> int:
        """Algorithmic size = the reference's planes.nbytes (bitplane.py:109-110)."""
        return self._width * words_needed(self._dim) * 8 * self._count

    @property
    def device_nbytes(self) -> int:
        """Bytes of the packed codes resident in HBM (0 after :meth:`release_codes`)."""
        return int(self._codes.numel()) if self._codes is not None else 0

    @property
    def codes(self):
        """torch.uint8 device buffer holding the bundle layout.  After :meth:`release_codes` it is rebuilt here, on the GPU,
        from the nibble layout (``xfbq_restore_codes_from_nibbles``) or the byte tiles (``xfbq_restore_codes_from_tiles``)."""
        if self._codes is None:
            torch = _native.require_cuda()
            L = _native.lib()
            src, fn = ((self._nibbles, L.xfbq_restore_codes_from_nibbles) if getattr(self, "_nibbles", None) is not None
                       else (getattr(self, "_tiles", None), L.xfbq_restore_codes_from_tiles))
            if src is None:  # release_layout() refuses to drop the last copy, so this cannot happen through the API
                raise NativeLibraryError("the packed codes were released and no derived layout is left to rebuild them from")
            with torch.cuda.device(src.device):
                codes = torch.zeros(max(int(L.xfbq_db_bytes(self._count, self._dim, self._width)), 16), dtype=torch.uint8, device=src.device)
                _native.check(fn(src.data_ptr(), self._count, self._dim, self._width, codes.data_ptr(), _stream_ptr(torch)))
            self._codes = codes
        return self._codes

    @property
    def device(self):
        """The GPU the codes live on (never rebuilds anything)."""
        for t in (self._codes, getattr(self, "_nibbles", None), getattr(self, "_tiles", None)):
            if t is not None:
                return t.device
        raise NativeLibraryError("no device buffer")

    @property
    def codes_ptr(self):
        """Device pointer of the packed codes, or None after :meth:`release_codes` (the scans that read a derived layout take a
        null pointer for them; nothing is rebuilt here)."""
        return self._codes.data_ptr() if self._codes is not None else None

    def release_codes(self) -> None:
        """Free the packed codes (the bundle layout) while a derived layout holds the same information: a server that only
        answers large batches then keeps the byte tiles alone (2x the packed size for 4-bit codes), one that only answers
        single queries the nibbles alone (1x).  Anything that reads bit planes (``planes``, ``batch_distances``, ``save_index``,
        the XOR/POPC kernels, building the other derived layout) rebuilds them on the GPU first."""
        if getattr(self, "_nibbles", None) is None and getattr(self, "_tiles", None) is None:
            raise InvalidInputError("no derived layout to rebuild the codes from: build nibble_layout or tile_layout first")
        self._codes = None

    @property
    def planes(self) -> np.ndarray:
        if self._planes is None:
            torch = _native.require_cuda()
            L = _native.lib()
            W64 = words_needed(self._dim)
            codes = self.codes
            with torch.cuda.device(codes.device):
                out = torch.zeros((self._width, W64, self._count), dtype=torch.int64, device=codes.device)
                if self._count:
                    _native.check(L.xfbq_bundles_to_planes(codes.data_ptr(), self._count, self._dim,
                                                           self._width, out.data_ptr(), _stream_ptr(torch)))
                host = out.cpu().numpy().view(np.uint64)
            host.setflags(write=False)
            self._planes = host
        return self._planes

    def _layout(self, attr: str, size_fn: str, build_fn: str, size_args):
        cached = getattr(self, attr, None)
        if cached is None:
            torch = _native.require_cuda()
            L = _native.lib()
            nbytes = int(getattr(L, size_fn)(*size_args))
            if nbytes == 0 or self._count == 0:
                return None
            codes = self.codes
            with torch.cuda.device(codes.device):
                cached = torch.empty(nbytes, dtype=torch.uint8, device=codes.device)
                _native.check(getattr(L, build_fn)(codes.data_ptr(), self._count, self._dim, self._width,
                                                   cached.data_ptr(), _stream_ptr(torch)))
            setattr(self, attr, cached)
        return cached

    @property
    def nibble_layout(self):
        """Derived row-major 4-bit copy of the codes (doc_bits <= 4, dim <= 512): what the mma.sync engine and the
        single-launch small-batch search stream (<= 16 queries, HBM-bound).  Built on the GPU on first use, cached; the
        same size as the packed codes for 4-bit codes.  None for shapes that engine does not take."""
        return self._layout("_nibbles", "xfbq_nibble_region_bytes", "xfbq_build_nibbles", (self._count, self._dim, self._width))

    @property
    def tile_layout(self):
        """Derived byte tiles (one code per byte, the shared-memory image of a tcgen05 B operand; dim <= 1024): what the
        tcgen05 engine streams (>= 17 queries).  Built on first use, cached; twice the packed size for 4-bit codes."""
        return self._layout("_tiles", "xfbq_tile_region_bytes", "xfbq_build_tiles", (self._count, self._dim))

    @property
    def derived_nbytes(self) -> dict:
        """Bytes of the derived layouts built so far (a server that only answers large batches never builds the nibbles,
        one that only answers single queries never builds the tiles)."""
        return {name: int(t.numel()) if t is not None else 0
                for name, t in (("nibbles", getattr(self, "_nibbles", None)), ("tiles", getattr(self, "_tiles", None)))}

    def release_layout(self, name: str) -> None:
        """Free a derived layout ("nibbles" or "tiles"); it is rebuilt if a later search needs it."""
        if name not in ("nibbles", "tiles"):
            raise InvalidInputError("layout must be 'nibbles' or 'tiles'")
        other = "_tiles" if name == "nibbles" else "_nibbles"
        if self._codes is None and getattr(self, other, None) is None:
            raise InvalidInputError("this layout is the only copy of the codes left (release_codes() was called): rebuild the codes first")
        setattr(self, "_" + name, None)

    def row(self, k: int) -> PackedVector:
        return PackedVector(np.ascontiguousarray(self.planes[:, :, k]), self._dim)

    def to_row_major(self) -> np.ndarray:
        return np.ascontiguousarray(self.planes.transpose(2, 0, 1))

    @classmethod
    def from_row_major(cls, rows, dim: int) -> "PackedMatrix":
        rows = np.asarray(rows, dtype=np.uint64)
        return cls(np.ascontiguousarray(rows.transpose(1, 2, 0)), dim)


def _as_float_matrix(values):
    """Host array as float32 or float64 without changing any value (the reference widens
    everything to float64, bitplane.py:229; float32 -> float64 is exact so float32 input is
    widened inside the kernel instead)."""
    a = np.asarray(values)
    if a.dtype == np.float32:
        return np.ascontiguousarray(a)
    return np.ascontiguousarray(a, dtype=np.float64)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def quantize_to_device(values, width: int, scale: float, queries: bool, defer_check: bool = False):
    """Run the quantizer kernel.  `values`: host array or CUDA tensor, (n, dim) f32/f64.
    Returns (device buffer, n, dim).  Raises InvalidInputError on non-finite scaled values
    (quant.py:142-143) exactly as the reference does.  With `defer_check` the device counter of
    non-finite values is returned as a fourth item instead of being read here (the read is a
    stream synchronisation): the caller enqueues the work that follows and checks it afterwards."""
    torch = _native.require_cuda()
    L = _native.lib()
    width = check_width(width)
    scale = float(scale)
    on_device = _is_torch(values)
    if on_device:
        if values.dtype not in (torch.float32, torch.float64):
            values = values.to(torch.float64)
        if not values.is_cuda:
            values = values.cuda(non_blocking=values.is_pinned())  # pinned: the host goes on to enqueue the kernels
        if values.stride(-1) != 1:
            values = values.contiguous()
        n, dim = values.shape
    else:
        values = _as_float_matrix(values)
        n, dim = values.shape
    if dim < 1:
        raise InvalidInputError("dim must be >= 1")
    # everything lives on the input's device (a CUDA tensor on a non-current device is quantized where it is)
    dev = values.device if on_device else torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        return _quantize_on(torch, L, dev, values, n, dim, width, scale, queries, on_device, defer_check)


def _quantize_on(torch, L, dev, values, n, dim, width, scale, queries, on_device, defer_check):
    st = _stream_ptr(torch)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    if queries:
        out = torch.empty(max(int(L.xfbq_query_bytes(n, dim, width)), 16) // 4, dtype=torch.int32, device=dev)
    else:
        out = torch.empty(max(int(L.xfbq_db_bytes(n, dim, width)), 16), dtype=torch.uint8, device=dev)
    row_bytes_out = int(L.xfbq_query_bytes(1, dim, width)) if queries else None

    def run(chunk, row0):
        f32 = chunk.dtype == torch.float32
        if queries:
            fn = L.xfbq_quantize_queries_f32 if f32 else L.xfbq_quantize_queries_f64
            dst = out.data_ptr() + row0 * row_bytes_out
        else:
            fn = L.xfbq_quantize_pack_f32 if f32 else L.xfbq_quantize_pack_f64
            dst = out.data_ptr() + int(L.xfbq_db_bytes(row0, dim, width))  # row0 is a multiple of 32
        ld = chunk.stride(0) if chunk.shape[0] > 1 else dim
        _native.check(fn(chunk.data_ptr(), chunk.shape[0], dim, ld, scale, width, dst,
                         bad.data_ptr(), st))

    if on_device:
        if n:
            run(values, 0)
    else:
        for row0 in range(0, n, _ROW_CHUNK):
            chunk = torch.from_numpy(values[row0:row0 + _ROW_CHUNK]).to(dev)
            run(chunk, row0)
            del chunk
    if defer_check:
        return out, n, dim, bad
    if n and int(bad.item()):
        raise InvalidInputError("cannot quantize non-finite values")
    return out, n, dim


def quantize_matrix(values, width: int, scale: float = 1.0) -> PackedMatrix:
    """Scale, quantize and pack an (n, dim) float matrix (bitplane.py:225-233) on the GPU."""
    if scale <= 0:
        raise InvalidInputError(f"scale must be positive, got {scale}")
    if not _is_torch(values):
        values = np.asarray(values)
    if values.ndim != 2:
        raise InvalidInputError("quantize_matrix expects an (n, dim) matrix")
    codes, n, dim = quantize_to_device(values, width, scale, queries=False)
    return PackedMatrix(None, dim, _codes=codes, _count=n, _width=check_width(width))


def quantize_queries(values, width: int, scale: float = 1.0, defer_check: bool = False):
    """Batched query quantizer: (nq, dim) -> device int32 buffer in the query layout
    (defer_check: -> (buffer, device counter of non-finite values), see quantize_to_device)."""
    if scale <= 0:
        raise InvalidInputError(f"scale must be positive, got {scale}")
    if values.ndim != 2:
        raise InvalidInputError("quantize_queries expects an (nq, dim) matrix")
    if defer_check:
        out, _, _, bad = quantize_to_device(values, width, scale, queries=True, defer_check=True)
        return out, bad
    out, _, _ = quantize_to_device(values, width, scale, queries=True)
    return out


def quantize_vector(values, width: int, scale: float = 1.0) -> PackedVector:
    """Scale, quantize and pack one float vector (bitplane.py:214-222) on the GPU."""
    if scale <= 0:
        raise InvalidInputError(f"scale must be positive, got {scale}")
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 1:
        raise InvalidInputError("quantize_vector expects a 1-D vector")
    width = check_width(width)
    if v.shape[0] == 0:
        return PackedVector(np.zeros((width, 0), dtype=np.uint64), 0)
    out, _, dim = quantize_to_device(v[None, :], width, scale, queries=True)
    C = (dim + 127) // 128
    words = out[: width * 4 * C].cpu().numpy().view(np.uint64).reshape(width, 2 * C)
    return PackedVector(np.ascontiguousarray(words[:, : words_needed(dim)]), dim)


def pack_matrix(codes, width: int) -> PackedMatrix:
    """(n, dim) uint codes -> PackedMatrix (bitplane.py:196-201).  Host bit packing of
    already-quantized codes is a format conversion, done with numpy and uploaded."""
    width = check_width(width)
    arr = np.asarray(codes)
    if arr.ndim != 2:
        raise InvalidInputError("pack_matrix expects an (n, dim) code array")
    if arr.size and int(arr.max()) >= (1 << width):
        raise InvalidInputError(f"code values exceed {width} bits")
    arr = arr.astype(np.uint8)
    n, dim = arr.shape
    nwords = words_needed(dim)
    planes = np.zeros((width, n, nwords * 8), dtype=np.uint8)
    for b in range(width):
        packed = np.packbits((arr >> b) & 1, axis=1, bitorder="little")
        planes[b, :, : packed.shape[1]] = packed
    planes = planes.view("<u8").astype(np.uint64, copy=False)
    return PackedMatrix(np.ascontiguousarray(planes.transpose(0, 2, 1)), dim)


def unpack_matrix(packed: PackedMatrix) -> np.ndarray:
    """Inverse of pack_matrix: (n, dim) uint8 codes (bitplane.py:204-211)."""
    planes = packed.planes
    n, dim = packed.count, packed.dim
    codes = np.zeros((n, dim), dtype=np.uint8)
    for b in range(packed.width):
        words = np.ascontiguousarray(planes[b].T).astype("<u8", copy=False)
        bits = np.unpackbits(words.view(np.uint8).reshape(n, -1), axis=1, bitorder="little")[:, :dim]
        codes |= (bits << b).astype(np.uint8)
    return codes
