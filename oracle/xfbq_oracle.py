"""CPU oracle for the XFBQ hot path -- TEST INFRASTRUCTURE, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  Nothing under
``paper_2008_02002_b200/`` imports it (tests/test_abi.py::test_product_never_imports_oracle enforces that).

Two independent restatements of the reference algorithm live here:

* ``np_*``  -- plain numpy, written from the reference's definitions;
* ``c_*``   -- ctypes bindings of ``oracle/xfbq_oracle.c`` (gcc -O3, OpenMP over
  queries), used for sizes where numpy is too slow and as the timed CPU baseline.

Parity is PINNED: ``oracle/gen_golden.py`` ran the unmodified reference
(``/root/reference/pkg/src/xfbq``) in the build container and committed its outputs
under ``tests/golden``; ``tests/test_oracle_golden.py`` checks both restatements
against those fixtures and the reference's worked examples.

Reference citations are paths under ``/root/reference/pkg/src/xfbq``.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "libxfbq_oracle.so"
_INFO = _HERE / "libxfbq_oracle.buildinfo"
_SRC = _HERE / "xfbq_oracle.c"

# --------------------------------------------------------------------------- numpy


def words_needed(dim: int) -> int:
    """bitplane.py:29-30."""
    return (int(dim) + 63) // 64


def distance_upper_bound(dim: int, wx: int, wy: int) -> int:
    """distance.py:25-29."""
    return int(dim) * ((1 << wx) - 1) * ((1 << wy) - 1)


def np_quantize_values(values, width: int) -> np.ndarray:
    """quant.py:138-148: odd = 2*floor(x*2^(w-1))+1, clip to +-(2^w-1), code=(hi-odd)/2."""
    x = np.asarray(values, dtype=np.float64)
    if not np.isfinite(x).all():
        raise ValueError("cannot quantize non-finite values")
    hi = float(2**width - 1)
    with np.errstate(over="ignore"):
        steps = np.floor(x * float(2 ** (width - 1)))
        odd = steps + steps + 1.0
    odd = np.minimum(np.maximum(odd, -hi), hi)
    return ((hi - odd) / 2.0).astype(np.uint8)


def np_pack_code_matrix(codes: np.ndarray, width: int) -> np.ndarray:
    """bitplane.py:151-163: (n, dim) u8 -> (width, words, n) u64, LE bit order, zero pad."""
    codes = np.asarray(codes, dtype=np.uint8)
    n, dim = codes.shape
    nwords = words_needed(dim)
    planes = np.zeros((width, nwords, n), dtype=np.uint64)
    cols = np.arange(dim)
    word_of = cols // 64
    shift_of = (cols % 64).astype(np.uint64)
    for b in range(width):
        bits = ((codes >> b) & 1).astype(np.uint64) << shift_of[None, :]  # (n, dim)
        for w in range(nwords):
            sel = word_of == w
            planes[b, w, :] = np.bitwise_or.reduce(bits[:, sel], axis=1) if sel.any() else 0
    return planes


def np_quantize_matrix(values, width: int, scale: float = 1.0) -> np.ndarray:
    """bitplane.py:225-233: widen to f64, multiply by float(scale), quantize, pack."""
    m = np.asarray(values, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError("expected (n, dim)")
    return np_pack_code_matrix(np_quantize_values(m * float(scale), width), width)


def np_quantize_vector(values, width: int, scale: float = 1.0) -> np.ndarray:
    """bitplane.py:214-222 -> (width, words) u64."""
    v = np.asarray(values, dtype=np.float64)
    return np_quantize_matrix(v[None, :], width, scale)[:, :, 0]


def np_unpack_codes(planes: np.ndarray, dim: int) -> np.ndarray:
    """Inverse of the pack (bitplane.py:204-211): (width, words, n) -> (n, dim) u8."""
    width, nwords, n = planes.shape
    codes = np.zeros((n, dim), dtype=np.uint8)
    for k in range(dim):
        w, s = divmod(k, 64)
        for b in range(width):
            codes[:, k] |= (((planes[b, w, :] >> np.uint64(s)) & np.uint64(1)) << b).astype(np.uint8)
    return codes


def _popcount64(a: np.ndarray) -> np.ndarray:
    """popcount.py:18-33 (SWAR form, independent of np.bitwise_count)."""
    a = a.astype(np.uint64, copy=True)
    m1, m2, m4 = np.uint64(0x5555555555555555), np.uint64(0x3333333333333333), np.uint64(0x0F0F0F0F0F0F0F0F)
    a = a - ((a >> np.uint64(1)) & m1)
    a = (a & m2) + ((a >> np.uint64(2)) & m2)
    a = (a + (a >> np.uint64(4))) & m4
    return (a * np.uint64(0x0101010101010101)) >> np.uint64(56)


def np_batch_distances(doc_planes: np.ndarray, query_planes: np.ndarray) -> np.ndarray:
    """_kernels.py:29-41 / :56-69: sum_{i,j,w} popcount(D[i,w,:] ^ Q[j,w]) << (i+j)."""
    wd, nwords, n = doc_planes.shape
    wq = query_planes.shape[0]
    out = np.zeros(n, dtype=np.uint64)
    for i in range(wd):
        for j in range(wq):
            for w in range(nwords):
                out += _popcount64(doc_planes[i, w] ^ query_planes[j, w]) << np.uint64(i + j)
    return out


def np_topk(dists: np.ndarray, k: int, row_offset: int = 0):
    """search.py:129-131 on the no-originals branch (:159-172): (dist asc, id asc)."""
    n = dists.shape[0]
    kk = min(int(k), n)
    order = np.lexsort((np.arange(n), dists))[:kk]
    return dists[order].astype(np.uint64), order.astype(np.int64) + int(row_offset)


def np_search(doc_planes, query_planes_batch, k: int, row_offset: int = 0):
    """SURVEY 8c composition, one query at a time. query_planes_batch: (nq, wq, words)."""
    nq = query_planes_batch.shape[0]
    kk = min(int(k), doc_planes.shape[2])
    out_d = np.zeros((nq, kk), dtype=np.uint64)
    out_i = np.zeros((nq, kk), dtype=np.int64)
    for q in range(nq):
        d = np_batch_distances(doc_planes, query_planes_batch[q])
        out_d[q], out_i[q] = np_topk(d, kk, row_offset)
    return out_d, out_i


def np_decode_inner_product_values(d, dim: int, wx: int, wy: int) -> np.ndarray:
    """distance.py:77-83: (hi - 2d) / 2^(wx+wy) in float64."""
    hi = float(distance_upper_bound(dim, wx, wy))
    return (hi - 2.0 * np.asarray(d, dtype=np.float64)) / float(1 << (wx + wy))


# ------------------------------------------------------------------------------- C


def _cpu_tag() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return hashlib.sha1(line.encode()).hexdigest()[:16]
    except OSError:
        pass
    return "unknown"


def build(force: bool = False) -> Path:
    """Compile xfbq_oracle.c with gcc (-march=native, so rebuilt when the host CPU differs)."""
    tag = _cpu_tag() + ":" + hashlib.sha1(_SRC.read_bytes()).hexdigest()[:16]
    if not force and _SO.exists() and _INFO.exists() and _INFO.read_text().strip() == tag:
        return _SO
    cmd = ["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-fvisibility=hidden",
           "-shared", "-o", str(_SO), str(_SRC), "-lm"]
    subprocess.run(cmd, check=True, capture_output=True)
    _INFO.write_text(tag + "\n")
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(str(build()))
    i64, i32, vp, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
    lib.xo_quantize_values.restype = i64
    lib.xo_quantize_values.argtypes = [vp, i64, i32, vp]
    lib.xo_pack_code_matrix.restype = None
    lib.xo_pack_code_matrix.argtypes = [vp, i64, i64, i32, vp]
    for name in ("xo_quantize_matrix_f32", "xo_quantize_matrix_f64"):
        fn = getattr(lib, name)
        fn.restype = i64
        fn.argtypes = [vp, i64, i64, i64, dbl, i32, vp]
    lib.xo_batch_distances.restype = None
    lib.xo_batch_distances.argtypes = [vp, i32, i64, i64, vp, i32, vp]
    lib.xo_packed_distance.restype = ctypes.c_uint64
    lib.xo_packed_distance.argtypes = [vp, i32, vp, i32, i64]
    lib.xo_topk.restype = i64
    lib.xo_topk.argtypes = [vp, i64, i64, vp, vp]
    lib.xo_search.restype = i64
    lib.xo_search.argtypes = [vp, i32, i64, i64, vp, i64, i32, i64, i64, i32, vp, vp]
    lib.xo_max_threads.restype = i32
    lib.xo_max_threads.argtypes = []
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def c_max_threads() -> int:
    return int(_load().xo_max_threads())


def c_quantize_matrix(values: np.ndarray, width: int, scale: float = 1.0) -> np.ndarray:
    """(n, dim) f32 or f64 -> (width, words, n) u64 planes; raises on non-finite scaled values."""
    lib = _load()
    v = np.asarray(values)
    if v.dtype == np.float32:
        v = np.ascontiguousarray(v)
        fn = lib.xo_quantize_matrix_f32
    else:
        v = np.ascontiguousarray(v, dtype=np.float64)
        fn = lib.xo_quantize_matrix_f64
    n, dim = v.shape
    planes = np.empty((width, words_needed(dim), n), dtype=np.uint64)
    bad = fn(_ptr(v), n, dim, dim, float(scale), int(width), _ptr(planes))
    if bad:
        raise ValueError("cannot quantize non-finite values")
    return planes


def c_batch_distances(doc_planes: np.ndarray, query_planes: np.ndarray) -> np.ndarray:
    lib = _load()
    d = np.ascontiguousarray(doc_planes, dtype=np.uint64)
    q = np.ascontiguousarray(query_planes, dtype=np.uint64)
    wd, nwords, n = d.shape
    out = np.empty(n, dtype=np.uint64)
    lib.xo_batch_distances(_ptr(d), wd, nwords, n, _ptr(q), q.shape[0], _ptr(out))
    return out


def c_topk(dists: np.ndarray, k: int):
    lib = _load()
    d = np.ascontiguousarray(dists, dtype=np.uint64)
    kk = min(int(k), d.shape[0])
    out_d = np.empty(kk, dtype=np.uint64)
    out_i = np.empty(kk, dtype=np.int64)
    if kk:
        lib.xo_topk(_ptr(d), d.shape[0], kk, _ptr(out_d), _ptr(out_i))
    return out_d, out_i


def c_search(doc_planes: np.ndarray, query_planes_batch: np.ndarray, k: int,
             row_offset: int = 0, threads: int = 0):
    """Batched oracle: (wd, words, n) x (nq, wq, words) -> ([nq, kk] u64 dists, [nq, kk] i64 ids)."""
    lib = _load()
    d = np.ascontiguousarray(doc_planes, dtype=np.uint64)
    q = np.ascontiguousarray(query_planes_batch, dtype=np.uint64)
    wd, nwords, n = d.shape
    nq, wq, qwords = q.shape
    assert qwords == nwords
    kk = min(int(k), n)
    out_d = np.empty((nq, kk), dtype=np.uint64)
    out_i = np.empty((nq, kk), dtype=np.int64)
    if kk and nq:
        lib.xo_search(_ptr(d), wd, nwords, n, _ptr(q), nq, wq, kk, int(row_offset),
                      int(threads), _ptr(out_d), _ptr(out_i))
    return out_d, out_i


def synthetic_unit_rows(n: int, dim: int, seed: int) -> np.ndarray:
    """Same recipe as the reference generator (dataio.py:104-124): PCG64 normal(0, 1/sqrt(dim)),
    float64 row normalise, cast float32.  Bit-identical to generate_synthetic(n, dim, seed).data
    (checked in tests/test_oracle_golden.py against a golden hash)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    data = rng.normal(0.0, 1.0 / np.sqrt(dim), size=(n, dim))
    data /= np.linalg.norm(data, axis=1, keepdims=True)
    return data.astype(np.float32)


def estimate_scale(vectors: np.ndarray, percentile: float = 0.98) -> float:
    """index.py:123-138: 1 / quantile(|x|, p)."""
    return 1.0 / float(np.quantile(np.abs(np.asarray(vectors)), percentile))
