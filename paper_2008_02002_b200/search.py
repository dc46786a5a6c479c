"""K-select front end: `k_select` (reference search.py:188-232) and the batched
`search(index, queries, k) -> (scores, indices)` the north star adds.

`search` is defined as the per-query composition of reference calls:
    pq = quantize_vector(float64(q), query_bits, scale); d = batch_distances(packed, pq)
    order = lexsort((arange(n), d))[:min(k, n)]; scores, indices = d[order], order
and is computed by one fused scan+top-K kernel launch per query batch: no score matrix
reaches HBM.  Keys are (distance << 32 | row id), so ties resolve to the lower row id
(search.py:129-131).
"""
from __future__ import annotations

import threading

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .bitplane import PackedMatrix, _is_torch, _stream_ptr, quantize_queries, quantize_vector
from .distance import collect_candidates_device, decode_inner_product_values, distance_upper_bound
from .errors import DimensionMismatchError, InvalidInputError
from .index import Index

MAX_K = 4096          # XFBQ_MAX_K
_QUERY_BATCH = 16384  # queries per scan launch (bounds grid.y and the partial-result workspace)
SCAN_EVENTS = None    # bench hook: set to a list to collect (start, end) CUDA events around each scan launch


@dataclass(frozen=True)
class SearchRequest:
    """search.py:33-51."""

    query: np.ndarray
    k: int
    extra_distance: int = 0

    def __post_init__(self):
        query = np.ascontiguousarray(self.query, dtype=np.float64)
        object.__setattr__(self, "query", query)
        if query.ndim != 1:
            raise InvalidInputError("query must be a 1-D vector")
        if not np.all(np.isfinite(query)):
            raise InvalidInputError("query contains non-finite entries")
        if self.k < 1:
            raise InvalidInputError(f"k must be >= 1, got {self.k}")
        if self.extra_distance < 0:
            raise InvalidInputError(f"extra_distance must be >= 0, got {self.extra_distance}")


@dataclass(frozen=True)
class SearchResult:
    """search.py:54-67."""

    hits: list
    candidate_count: int
    threshold_distance: int
    approximate: bool = False
    stage_seconds: dict | None = field(default=None, compare=False)


_WORKSPACES = {}   # (device index, stream, host thread) -> uint8 tensor, grown on demand: the scans ONE thread enqueues on a stream are ordered and
                   # can share it; two host threads on the same stream interleave their launches, so each thread has its own
_NONFINITE = {}    # (device index, host thread) -> int64[1] counter of non-finite query values seen by that thread's fused small-batch searches


def _nf_key(torch, dev):
    return (dev.index if dev.index is not None else torch.cuda.current_device(), threading.get_ident())


def _workspace(torch, dev, nbytes: int):
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream, threading.get_ident())
    ws = _WORKSPACES.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=dev)
        _WORKSPACES[key] = ws
    return ws


def _search_small_fused(index: Index, queries, k: int, row_offset: int):
    """<= 16 float queries resident on the index's GPU: quantizer, threshold seeding, scan and merge in ONE cooperative launch
    (xfbq_search_small_*).  Returns (keys, counter of non-finite query values) or None when the shape takes the general path."""
    torch = _native.require_cuda()
    L = _native.lib()
    packed, p = index.packed, index.params
    nq = int(queries.shape[0])
    if not 1 <= nq <= 16 or packed.width > 4 or p.query_bits > 7 or packed.dim > 512 or k > 1024:
        return None
    dev = packed.device
    ws_bytes = int(L.xfbq_search_small_workspace_bytes(packed.count, packed.dim, packed.width, nq, p.query_bits, k))
    if ws_bytes <= 0:
        return None
    if queries.dtype not in (torch.float32, torch.float64):
        queries = queries.to(torch.float64)
    if queries.stride(-1) != 1 or queries.device != dev:
        queries = queries.to(dev).contiguous()
    nib = packed.nibble_layout
    if nib is None:
        return None
    counter = _NONFINITE.get(_nf_key(torch, dev))
    if counter is None:
        counter = _NONFINITE[_nf_key(torch, dev)] = torch.zeros(1, dtype=torch.int64, device=dev)
    keys = torch.empty((nq, k), dtype=torch.int64, device=dev)
    ws = _workspace(torch, dev, ws_bytes)
    fn = L.xfbq_search_small_f32 if queries.dtype == torch.float32 else L.xfbq_search_small_f64
    ld = queries.stride(0) if nq > 1 else packed.dim
    if SCAN_EVENTS is not None:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    _native.check(fn(packed.codes_ptr, nib.data_ptr(), packed.count, packed.dim, packed.width, queries.data_ptr(), nq, ld,
                     float(p.scale), p.query_bits, k, int(row_offset), keys.data_ptr(), counter.data_ptr(), ws.data_ptr(), ws.numel(),
                     _stream_ptr(torch)))
    if SCAN_EVENTS is not None:
        ev[1].record()
        SCAN_EVENTS.append(ev)
    return keys, counter


def _kselect_small_fused(index: Index, query: np.ndarray, k: int, extra: int, want_ids: bool, cap: int):
    """k_select's quantize + scan + top-k + histogram/gather stage as ONE cooperative launch (xfbq_kselect_small_f64).
    Returns (keys int64[k] on the host, candidate count, device ids or None), or None when the shape takes the general path or a
    candidate list had to be cut during the scan (large extra_distance, heavy ties): the caller then runs the separate passes."""
    torch = _native.require_cuda()
    L = _native.lib()
    packed, p = index.packed, index.params
    if packed.width > 4 or p.query_bits > 7 or packed.dim > 512 or k > 1024 or extra >= (1 << 30):
        return None
    dev = packed.device
    ws_bytes = int(L.xfbq_search_small_workspace_bytes(packed.count, packed.dim, packed.width, 1, p.query_bits, k))
    if ws_bytes <= 0:
        return None
    nib = packed.nibble_layout
    if nib is None:
        return None
    with torch.cuda.device(dev):
        counter = _NONFINITE.get(_nf_key(torch, dev))
        if counter is None:
            counter = _NONFINITE[_nf_key(torch, dev)] = torch.zeros(1, dtype=torch.int64, device=dev)
        q_dev = torch.from_numpy(np.ascontiguousarray(query, dtype=np.float64)[None, :]).to(dev)
        keys = torch.empty(k + 2, dtype=torch.int64, device=dev)        # k keys, candidate count, inexact flag: one D2H copy
        ids = torch.empty(cap if want_ids else 0, dtype=torch.int64, device=dev)
        ws = _workspace(torch, dev, ws_bytes)
        _native.check(L.xfbq_kselect_small_f64(packed.codes_ptr, nib.data_ptr(), packed.count, packed.dim, packed.width,
                                               q_dev.data_ptr(), 1, packed.dim, float(p.scale), p.query_bits, k, int(extra), 0,
                                               keys.data_ptr(), keys.data_ptr() + 8 * k, ids.data_ptr() if want_ids else None, cap,
                                               keys.data_ptr() + 8 * (k + 1), counter.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(torch)))
        (host,) = to_host_arrays(keys)
        raise_pending_nonfinite(dev)
    count, inexact = int(host[k]), int(host[k + 1]) & 0xFFFFFFFF
    if inexact or (want_ids and count > cap):
        return None
    return host[:k], count, (ids[:count] if want_ids else None)


def scan_topk_device(packed: PackedMatrix, qwords, nq: int, query_bits: int, k: int, row_offset: int = 0):
    """Launch the fused scan+top-K on device-resident query words (query layout).
    Returns an int64 CUDA tensor [nq, k] holding the uint64 keys bit-for-bit
    (distance << 32 | row_offset + row; 0xFFFF... for empty slots)."""
    torch = _native.require_cuda()
    L = _native.lib()
    dev = packed.device
    with torch.cuda.device(dev):
        keys = torch.empty((nq, k), dtype=torch.int64, device=dev)
        if nq == 0:
            return keys
        C = (packed.dim + 127) // 128
        words_per_query = query_bits * 4 * C  # int32 elements
        st = _stream_ptr(torch)
        if k > MAX_K:
            # Wider than the fused selector (XFBQ_MAX_K lists per query): the reference accepts any k (search.py:212), so
            # fall back to the distance kernel + a full device sort of the (distance << 32 | id) keys, one query at a time.
            # torch.sort is library code (CUB): this regime (k > 4096) is outside the fused hot path.
            ids = torch.arange(packed.count, dtype=torch.int64, device=dev) + int(row_offset)
            d = torch.empty(packed.count, dtype=torch.int64, device=dev)
            for qi in range(nq):
                _native.check(L.xfbq_batch_distances(packed.codes.data_ptr(), packed.count, packed.dim, packed.width,
                                                     qwords.data_ptr() + qi * words_per_query * 4, query_bits, d.data_ptr(), st))
                keys[qi] = torch.sort((d << 32) | ids).values[:k]
            return keys
        for q0 in range(0, nq, _QUERY_BATCH):
            qn = min(_QUERY_BATCH, nq - q0)
            # the derived layout the preferred plan reads is built on first use (tiles: tcgen05 engine; nibbles: mma.sync
            # engine); one that already exists is passed along too (the mma.sync path seeds its thresholds from tiles)
            want = int(L.xfbq_scan_layouts(packed.count, packed.dim, packed.width, qn, query_bits, k))
            nib = packed.nibble_layout if want & 2 else getattr(packed, "_nibbles", None)
            tiles = packed.tile_layout if want & 4 else getattr(packed, "_tiles", None)
            have = (2 if nib is not None else 0) | (4 if tiles is not None else 0)
            ws_bytes = int(L.xfbq_scan_workspace_bytes(packed.count, packed.dim, packed.width, qn, query_bits, k, have))
            if ws_bytes < 0:
                _native.check(_native.E_INVALID)
            ws = _workspace(torch, dev, max(ws_bytes, 16))
            qptr = qwords.data_ptr() + q0 * words_per_query * 4
            if SCAN_EVENTS is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            # the XOR/POPC kernels (want == 0) read the packed codes: rebuilt here if they were released; the other plans do not
            _native.check(L.xfbq_scan_topk_layouts(packed.codes.data_ptr() if want == 0 else packed.codes_ptr, nib.data_ptr() if nib is not None else None,
                                                   tiles.data_ptr() if tiles is not None else None, packed.count, packed.dim,
                                                   packed.width, qptr, qn, query_bits, k, int(row_offset),
                                                   keys.data_ptr() + q0 * k * 8, ws.data_ptr(), ws.numel(), st))
            if SCAN_EVENTS is not None:
                ev[1].record()
                SCAN_EVENTS.append(ev)
    return keys


def unpack_keys_device(keys):
    """int64 key tensor -> (distances int64, row ids int64) on the device (-1 for empty slots)."""
    torch = _native.require_cuda()
    L = _native.lib()
    with torch.cuda.device(keys.device):
        d = torch.empty_like(keys)
        i = torch.empty_like(keys)
        _native.check(L.xfbq_unpack_keys(keys.data_ptr(), keys.numel(), d.data_ptr(), i.data_ptr(),
                                         _stream_ptr(torch)))
    return d, i


def _check_queries(index: Index, queries):
    if queries.ndim != 2:
        raise InvalidInputError("queries must be an (nq, dim) matrix")
    if queries.shape[1] != index.params.dim:
        raise DimensionMismatchError(f"query dim {queries.shape[1]} != index dim {index.params.dim}")


def search_device(index: Index, queries, k: int, row_offset: int = 0, check: bool = True):
    """Batched search returning device tensors (keys int64 [nq, min(k, n)]).
    `queries`: host array or CUDA tensor (nq, dim), float32/float64.

    Non-finite queries raise InvalidInputError like the reference (quant.py:142-143).  Reading the quantizer's counter is a
    stream synchronisation; `check=False` skips it for asynchronous pipelines of small device-resident batches (the fused
    single-launch path): a query holding a non-finite value then comes back as empty keys (all ones) and
    `pending_nonfinite()` reports it at the caller's next synchronisation point."""
    if k < 1:
        raise InvalidInputError(f"k must be >= 1, got {k}")
    if not _is_torch(queries):
        queries = np.asarray(queries)
        if queries.dtype != np.float32:
            queries = np.ascontiguousarray(queries, dtype=np.float64)
    _check_queries(index, queries)
    p = index.params
    kk = min(int(k), index.n)
    torch = _native.require_cuda()
    dev = index.packed.device
    with torch.cuda.device(dev):
        if kk == 0 or queries.shape[0] == 0:
            return torch.empty((queries.shape[0], kk), dtype=torch.int64, device=dev)
        on_device = _is_torch(queries) and queries.is_cuda
        if queries.shape[0] <= 16:
            # small batches: one cooperative launch from the float queries (host queries are copied first)
            qt = queries
            if not on_device:
                qt = torch.from_numpy(np.ascontiguousarray(queries)) if not _is_torch(queries) else queries
                qt = qt.to(dev, non_blocking=qt.is_pinned())
            fused = _search_small_fused(index, qt, kk, row_offset)
            if fused is not None:
                keys, counter = fused
                if check or not on_device:
                    raise_pending_nonfinite(dev)
                return keys
        if on_device:
            # device-resident queries: the counter is read right after the quantizer, the scan runs asynchronously
            # (back-to-back searches overlap their launches with the previous scan: 358 vs 396 us per single query)
            qwords = quantize_queries(queries, p.query_bits, p.scale)
            return scan_topk_device(index.packed, qwords, queries.shape[0], p.query_bits, kk, row_offset)
        # host queries (the caller waits for host results anyway): copy, quantizer and scan are enqueued back to back
        # and the non-finite counter is read afterwards -- the read synchronises the stream; no result is returned
        # when the reference would have raised (quant.py:142-143)
        qwords, bad = quantize_queries(queries, p.query_bits, p.scale, defer_check=True)
        keys = scan_topk_device(index.packed, qwords, queries.shape[0], p.query_bits, kk, row_offset)
        if int(bad.item()):
            raise InvalidInputError("cannot quantize non-finite values")
        return keys


def pending_nonfinite(device=None) -> int:
    """Non-finite query values the calling thread's fused small-batch searches on `device` have met since the last check (synchronises)."""
    torch = _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    counter = _NONFINITE.get(_nf_key(torch, dev))
    return int(counter.item()) if counter is not None else 0


def raise_pending_nonfinite(device=None) -> None:
    """Raise InvalidInputError (and clear the counter) if a fused small-batch search on `device` met a non-finite query."""
    if pending_nonfinite(device):
        torch = _native.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        _NONFINITE[_nf_key(torch, dev)].zero_()
        raise InvalidInputError("cannot quantize non-finite values")


def search(index: Index, queries, k: int):
    """Exhaustive top-k for a batch of float queries.

    Returns ``(scores, indices)``: int64 arrays [nq, min(k, n)]; ``scores`` are the integer
    XOR/popcount distances (smaller = more similar), rows ordered by (distance asc, row id
    asc).  Host arrays (numpy, or pinned/pageable CPU tensors) in -> numpy out, with one H2D
    copy of the queries and one D2H copy of the results; CUDA tensors in -> CUDA tensors out."""
    keys = search_device(index, queries, k)
    d, i = unpack_keys_device(keys)
    if _is_torch(queries) and queries.is_cuda:
        return d, i
    return to_host_arrays(d, i)


def to_host_arrays(*tensors):
    """Device tensors -> numpy arrays through pinned staging buffers (torch's caching host allocator
    recycles them), all copies in flight together, one stream synchronisation."""
    torch = _native.require_cuda()
    if not tensors:
        return ()
    with torch.cuda.device(tensors[0].device):
        host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in tensors]
        for h, t in zip(host, tensors):
            h.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    return tuple(h.numpy() for h in host)


def _refine_device(index: Index, query: np.ndarray, cand, k: int):
    """refine with originals (search.py:153-157 + _rank_hits :129-131): float64 dot products of the candidates' float32
    rows with the query and the k best by (similarity desc, id asc), in xfbq_refine_f32 (gather-dot kernel + bounded
    block top-k).  `cand`: device int64 row ids, any order.  Originals that live in HBM (CUDA tensor: build_index from a
    CUDA tensor, or Index.originals_to_device()) are gathered by the kernel; host-resident originals are gathered on the
    host (count rows, a memory move) and only those rows are uploaded -- the whole matrix (10 GB at 10M x 256) never is."""
    torch = _native.require_cuda()
    L = _native.lib()
    dev = index.packed.device
    count = int(cand.numel())
    kk = min(int(k), count)
    if kk == 0:
        return []
    orig = getattr(index, "_originals_dev", None)
    if orig is None and _is_torch(index.originals) and index.originals.is_cuda:
        orig = index.originals
    with torch.cuda.device(dev):
        st = _stream_ptr(torch)
        q_dev = torch.from_numpy(np.ascontiguousarray(query, dtype=np.float64)).to(dev)
        if orig is not None:
            rows, gathered, n_rows = orig, 0, index.n
        else:
            ids_host = cand.cpu().numpy()
            host_rows = index.originals.numpy() if _is_torch(index.originals) else np.asarray(index.originals)
            rows = torch.from_numpy(np.ascontiguousarray(host_rows[ids_host], dtype=np.float32)).to(dev)
            gathered, n_rows = 1, count
        if rows.dtype != torch.float32 or rows.stride(-1) != 1:
            rows = rows.to(torch.float32).contiguous()
        if kk > MAX_K:
            # library fallback beyond XFBQ_MAX_K (no hand-written selector that wide): float64 GEMV + two stable sorts
            sel_rows = rows if gathered else rows[cand]
            sims = sel_rows.to(torch.float64) @ q_dev
            by_id = torch.sort(cand, stable=True)
            by_sim = torch.sort(-sims[by_id.indices], stable=True)
            order = by_id.indices[by_sim.indices][:kk]
            sims_out, ids_out = sims[order], cand[order]
        else:
            ws_bytes = int(L.xfbq_refine_workspace_bytes(count, kk))
            ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
            sims_out = torch.empty(kk, dtype=torch.float64, device=dev)
            ids_out = torch.empty(kk, dtype=torch.int64, device=dev)
            ld = rows.stride(0) if rows.shape[0] > 1 else rows.shape[1]
            _native.check(L.xfbq_refine_f32(rows.data_ptr(), n_rows, rows.shape[1], ld, gathered, cand.data_ptr(), count,
                                            q_dev.data_ptr(), kk, sims_out.data_ptr(), ids_out.data_ptr(), ws.data_ptr(),
                                            ws_bytes, st))
        sims_h, ids_h = to_host_arrays(sims_out, ids_out)
    return [(int(i), float(s)) for i, s in zip(ids_h, sims_h)]


def k_select(index: Index, request: SearchRequest, collect_timing: bool = False) -> SearchResult:
    """search.py:188-232, one query.  Without originals the hits come straight from the fused
    scan+top-K (ranking by quantized similarity, `approximate=True`); with originals the
    candidates d <= kth + extra are re-ranked by float64 dot products on the device."""
    p = index.params
    if request.query.shape[0] != p.dim:
        raise DimensionMismatchError(f"query dim {request.query.shape[0]} != index dim {p.dim}")
    timings = {} if collect_timing else None
    if index.n == 0:
        return SearchResult(hits=[], candidate_count=0, threshold_distance=0,
                            approximate=index.originals is None, stage_seconds=timings)
    torch = _native.require_cuda()
    sync = torch.cuda.synchronize if collect_timing else (lambda: None)
    kk = min(request.k, index.n)
    upper = distance_upper_bound(p.dim, p.doc_bits, p.query_bits)

    t0 = time.perf_counter()
    dev = index.packed.device
    want_ids = index.originals is not None
    extra = min(int(request.extra_distance), upper)
    fused = _kselect_small_fused(index, request.query, kk, extra, want_ids, cap=max(1 << 16, 4 * kk))
    if fused is not None:
        # one cooperative launch did the whole of search.py:206-214: quantize, distances + top-k, threshold, candidate gather
        host_keys, candidate_count, cand = fused
        kn = host_keys.view(np.uint64)
        top_d, top_i = (kn >> np.uint64(32)).astype(np.int64), (kn & np.uint64(0xFFFFFFFF)).astype(np.int64)
        threshold = int(top_d[kk - 1]) + int(request.extra_distance)
        t1, t2 = t0, time.perf_counter()   # the fused launch is booked under "distances"
    else:
        # the query never round-trips through the host: upload the floats, quantize on the device (counter read after the scan)
        with torch.cuda.device(dev):
            q_dev = torch.from_numpy(request.query[None, :]).to(dev)
            qwords, bad = quantize_queries(q_dev, p.query_bits, p.scale, defer_check=True)
        sync(); t1 = time.perf_counter()
        keys = scan_topk_device(index.packed, qwords, 1, p.query_bits, kk)
        top_d, top_i = to_host_arrays(*(t[0] for t in unpack_keys_device(keys)))
        if int(bad.item()):
            raise InvalidInputError("cannot quantize non-finite values")
        sync(); t2 = time.perf_counter()
        # the k-th smallest distance IS the reference's histogram threshold (search.py:206-213); the gather is one
        # more pass over the codes (no distance array): count, and row ids when they are re-ranked
        threshold = int(top_d[kk - 1]) + int(request.extra_distance)
        candidate_count, cand = collect_candidates_device(index.packed, qwords, min(threshold, upper), want_ids=want_ids,
                                                          cap=max(1 << 16, 4 * kk), query_bits=p.query_bits)
    sync(); t3 = time.perf_counter()
    if index.originals is None:
        sims = decode_inner_product_values(top_d, p.dim, p.doc_bits, p.query_bits)
        sims /= p.scale * p.scale                                       # search.py:167-171
        hits = [(int(i), float(s)) for i, s in zip(top_i, sims)]
        approximate = True
    else:
        hits = _refine_device(index, request.query, cand, request.k)
        approximate = False
    sync(); t4 = time.perf_counter()
    if index.ids is not None:
        hits = [(int(index.ids[row]), sim) for row, sim in hits]
    if collect_timing:
        timings["quantize_query"] = t1 - t0
        timings["distances"] = t2 - t1
        timings["histogram_gather"] = t3 - t2
        timings["refine"] = t4 - t3
    return SearchResult(hits=hits, candidate_count=candidate_count, threshold_distance=threshold,
                        approximate=approximate, stage_seconds=timings)


# ------------------------------------------------------------------------------------------------------------------
# Stand-alone stages of the reference pipeline (search.py:70-185), for callers that use them directly.  k_select above
# fuses them: it never builds a distance array, a histogram or an id list of the whole database.
def _device_int64(distances):
    """Distance array (numpy uint64/int64 or CUDA int64 tensor) -> CUDA int64 tensor."""
    torch = _native.require_cuda()
    if _is_torch(distances):
        t = distances if distances.is_cuda else distances.cuda()
        return t.to(torch.int64).contiguous().reshape(-1)
    a = np.asarray(distances)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64).reshape(-1)).cuda()


@dataclass(frozen=True)
class DistanceHistogram:
    """search.py:68-98: frequency of every integer distance value in 0..upper_bound (bins: host int64 array)."""

    bins: np.ndarray

    @classmethod
    def from_distances(cls, distances, upper_bound: int) -> "DistanceHistogram":
        torch = _native.require_cuda()
        L = _native.lib()
        d = _device_int64(distances)
        if d.numel() == 0:
            raise InvalidInputError("cannot histogram an empty distance array")
        nbins = int(upper_bound) + 1
        with torch.cuda.device(d.device):
            hist = torch.empty(nbins, dtype=torch.int64, device=d.device)
            over = torch.empty(1, dtype=torch.int64, device=d.device)
            _native.check(L.xfbq_distance_histogram(d.data_ptr(), d.numel(), nbins, hist.data_ptr(), over.data_ptr(), _stream_ptr(torch)))
            if int(over.item()):
                raise InvalidInputError(f"distance {int(d.max())} exceeds upper bound {upper_bound}")
            return cls(bins=hist.cpu().numpy())

    @property
    def total(self) -> int:
        return int(self.bins.sum())

    def kth_smallest(self, k: int) -> int:
        """Smallest distance value t with at least k distances <= t."""
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        torch = _native.require_cuda()
        L = _native.lib()
        k = min(int(k), self.total)
        hist = torch.from_numpy(np.ascontiguousarray(self.bins, dtype=np.int64)).cuda()
        out = torch.empty(1, dtype=torch.int64, device=hist.device)
        _native.check(L.xfbq_histogram_kth(hist.data_ptr(), hist.numel(), max(k, 1), out.data_ptr(), _stream_ptr(torch)))
        return int(out.item())


def histogram_kth_distance(distances, k: int, extra: int = 0, upper_bound: int | None = None) -> int:
    """search.py:101-117: k-th smallest distance by histogram, plus `extra`."""
    d = _device_int64(distances)
    if d.numel() == 0:
        raise InvalidInputError("cannot select from an empty distance array")
    if extra < 0:
        raise InvalidInputError(f"extra must be >= 0, got {extra}")
    if upper_bound is None:
        upper_bound = int(d.max())
    return DistanceHistogram.from_distances(d, upper_bound).kth_smallest(k) + int(extra)


def gather_candidates(distances, threshold: int) -> np.ndarray:
    """search.py:120-126: ids with distance <= threshold, ascending (ordered compaction on the GPU)."""
    torch = _native.require_cuda()
    L = _native.lib()
    d = _device_int64(distances)
    if d.numel() == 0 or threshold < 0:
        return np.empty(0, dtype=np.int64)
    n = d.numel()
    with torch.cuda.device(d.device):
        ws = torch.empty(int(L.xfbq_gather_workspace_bytes(n)) // 8, dtype=torch.int64, device=d.device)
        st = _stream_ptr(torch)
        _native.check(L.xfbq_gather_le_count(d.data_ptr(), n, int(threshold), ws.data_ptr(), ws.numel() * 8, st))
        count = int(ws[(n + 65535) // 65536].item())
        ids = torch.empty(count, dtype=torch.int64, device=d.device)
        if count:
            _native.check(L.xfbq_gather_le_ids(d.data_ptr(), n, int(threshold), ws.data_ptr(), ids.data_ptr(), st))
        return ids.cpu().numpy()


def refine(index: Index, query, candidates, k: int, distances=None):
    """search.py:134-172: re-rank candidate rows; returns (hits, approximate).  With originals: float64 dot products of the
    float32 rows (xfbq_refine_f32); without: similarities decoded from quantized distances, flagged approximate."""
    torch = _native.require_cuda()
    cand = np.asarray(candidates, dtype=np.int64)
    if cand.size == 0:
        return [], index.originals is None
    q = np.ascontiguousarray(query, dtype=np.float64)
    p = index.params
    if index.originals is not None:
        hits = _refine_device(index, q, torch.from_numpy(cand).to(index.packed.device), k)
        return hits, False
    if distances is None:
        from .distance import batch_distances_device
        cand_d = batch_distances_device(index.packed, quantize_vector(q, p.query_bits, p.scale))[torch.from_numpy(cand).to(index.packed.device)].cpu().numpy()
    else:
        cand_d = np.asarray(distances)[cand]
    sims = decode_inner_product_values(cand_d, p.dim, p.doc_bits, p.query_bits)
    sims /= p.scale * p.scale
    order = np.lexsort((cand, -sims))[:k]                               # search.py:129-131 on <= candidate-count values
    return [(int(cand[i]), float(sims[i])) for i in order], True


def suggest_extra_distance(index: Index, fraction: float) -> int:
    """search.py:175-185."""
    if not 0.0 <= fraction <= 1.0:
        raise InvalidInputError(f"fraction must be in [0, 1], got {fraction}")
    p = index.params
    return round(fraction * distance_upper_bound(p.dim, p.query_bits, p.doc_bits))
