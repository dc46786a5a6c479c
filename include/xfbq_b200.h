/*
 * xfbq_b200.h -- C ABI of the B200-native XFBQ hot path (libxfbq_b200.so).
 *
 * The reference (arXiv 2008.02002 package `xfbq`, pure Python) has no FFI; its
 * narrowest swap point is the callable `batch_distances_kernel(doc_planes,
 * query_planes, out)` (pkg/src/xfbq/_kernels.py:71-75).  The entry points below
 * are what a binding for the hot path quantize -> pack -> XOR/POPC scan ->
 * top-K -> merge would call; each cites the reference code it replaces.
 * INTEGRATION.md shows the ctypes stub a maintainer of the reference would add.
 *
 * Conventions
 *   - every pointer named *_dev is a CUDA device pointer owned by the caller; the
 *     library never allocates or frees device memory and keeps no global state
 *     besides a thread-local error string;
 *   - `stream` is a cudaStream_t passed as void* (NULL = default stream); all
 *     work is enqueued asynchronously on it, calls are re-entrant per
 *     (stream, workspace);
 *   - return value: 0 = ok, nonzero = error (XFBQ_E_*), message via
 *     xfbq_last_error() (thread-local, valid until the next failing call);
 *   - no exceptions cross the boundary, no torch types appear in signatures.
 *
 * Device layouts
 *   bundle layout (database codes): documents are grouped in bundles of 32
 *     ("32-doc warp bundles"); C = ceil(dim/128) 128-bit chunks per
 *     plane; element (bundle b, plane i, chunk c, lane l) is one 16-byte word
 *     at index ((b*width + i)*C + c)*32 + l holding dims [128c, 128c+128) of
 *     bit-plane i of document 32b+l, little-endian bit order (dimension k ->
 *     bit k%32 of 32-bit word (k%128)/32), identical bit numbering to the
 *     reference's uint64 words (bitplane.py:1-9).  Padding dims and padding
 *     documents are all-zero bits.  Size: xfbq_db_bytes().
 *   query layout: uint32 [nq][width][4*C], same bit numbering, zero padded.
 *   keys: uint64 (distance << 32) | global_row_id ; ascending key order is the
 *     reference's ranking (distance asc, row id asc; search.py:129-131).
 *     Unused slots hold UINT64_MAX.
 */
#ifndef XFBQ_B200_H
#define XFBQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XFBQ_ABI_VERSION 1

#define XFBQ_OK 0
#define XFBQ_E_INVALID 1     /* argument violates a precondition (InvalidInputError) */
#define XFBQ_E_CUDA 2        /* CUDA runtime error */
#define XFBQ_E_UNSUPPORTED 3 /* shape outside what the kernels implement */

#define XFBQ_MAX_WIDTH 8     /* quant.py:20 MAX_WIDTH */
#define XFBQ_MAX_K 4096      /* largest k one scan pass selects */

int xfbq_abi_version(void);
const char *xfbq_last_error(void);

/* bitplane.py:29-30 words_needed, in 128-bit chunks */
int64_t xfbq_chunks128(int64_t dim);
/* bytes of the bundle layout for n documents (n rounded up to 32) */
int64_t xfbq_db_bytes(int64_t n, int64_t dim, int width);
/* bytes of the query layout */
int64_t xfbq_query_bytes(int64_t nq, int64_t dim, int width);
/* distance.py:25-29 distance_upper_bound */
int64_t xfbq_distance_upper_bound(int64_t dim, int width_x, int width_y);

/*
 * Quantizer + bit-plane packer: replaces quantize_matrix (bitplane.py:225-233) =
 * widen to float64, multiply by `scale`, quantize_values (quant.py:138-148),
 * _pack_code_matrix (bitplane.py:151-163).  x_dev is row-major (n, dim) with
 * leading dimension ld (elements).  *nonfinite_dev (device uint64, caller
 * zeroes it) is incremented by the number of non-finite scaled values; the
 * reference raises InvalidInputError when that is nonzero (quant.py:142-143).
 * Output: bundle layout.
 */
int xfbq_quantize_pack_f32(const float *x_dev, int64_t n, int64_t dim, int64_t ld, double scale,
                           int width, void *db_out_dev, uint64_t *nonfinite_dev, void *stream);
int xfbq_quantize_pack_f64(const double *x_dev, int64_t n, int64_t dim, int64_t ld, double scale,
                           int width, void *db_out_dev, uint64_t *nonfinite_dev, void *stream);
/* Same arithmetic for queries (quantize_vector, bitplane.py:214-222); output: query layout. */
int xfbq_quantize_queries_f32(const float *q_dev, int64_t nq, int64_t dim, int64_t ld,
                              double scale, int width, uint32_t *q_out_dev,
                              uint64_t *nonfinite_dev, void *stream);
int xfbq_quantize_queries_f64(const double *q_dev, int64_t nq, int64_t dim, int64_t ld,
                              double scale, int width, uint32_t *q_out_dev,
                              uint64_t *nonfinite_dev, void *stream);

/*
 * Layout conversion between the reference's PackedMatrix.planes
 * ((width, ceil(dim/64), n) uint64, bitplane.py:79-81) and the bundle layout.
 */
int xfbq_planes_to_bundles(const uint64_t *planes_dev, int64_t n, int64_t dim, int width,
                           void *db_out_dev, void *stream);
int xfbq_bundles_to_planes(const void *db_dev, int64_t n, int64_t dim, int width,
                           uint64_t *planes_out_dev, void *stream);

/*
 * Derived layouts for the tensor-core engines (doc_bits <= 4), one buffer of xfbq_nibble_bytes(n, dim)
 * bytes filled by xfbq_planes_to_nibbles from the bundle layout on the GPU:
 *   [nibble layout] row-major 4-bit codes, 64*C bytes per document (documents rounded up to 32), one
 *                   16-byte word per group of 32 dims whose 32-bit word e holds in nibble m the code of
 *                   dimension 4m + e (streamed by the mma.sync engine: <= 16 queries, HBM-bound);
 *   [byte tiles]    (any doc_bits 1..8, dim <= 1024) tiles of 128 documents x 128*C bytes, one code per byte,
 *                   K-major with the 128-byte swizzle: the exact shared-memory image of a tcgen05.mma B operand,
 *                   copied by one cp.async.bulk per tile (streamed by the tcgen05 engine: >= 17 queries, and every
 *                   batch size where the mma.sync engine does not go: doc_bits > 4 or dim > 512).
 * The tile region starts at the nibble region's size rounded up to 1024 bytes.
 */
/* The two layouts can also be built and passed separately (a batch server needs only the tiles: 2x the packed size for 4-bit
 * codes; a low-latency server only the nibbles: 1x): */
#define XFBQ_LAYOUT_NIBBLES 2
#define XFBQ_LAYOUT_TILES 4
int64_t xfbq_nibble_region_bytes(int64_t n, int64_t dim, int width);  /* 0 when the mma.sync engine does not take the shape */
int64_t xfbq_tile_region_bytes(int64_t n, int64_t dim);               /* 0 for dim > 1024 */
int xfbq_build_nibbles(const void *db_dev, int64_t n, int64_t dim, int width, void *nibbles_out_dev, void *stream);
int xfbq_build_tiles(const void *db_dev, int64_t n, int64_t dim, int width, void *tiles_out_dev, void *stream);
/* The inverse conversions: rebuild the packed codes (bundle layout, xfbq_db_bytes) from a derived layout, so that a server may
 * free them while it only scans (a batch server then holds the tiles alone, 2x the packed size for 4-bit codes; a single-query
 * server the nibbles alone, 1x) and get them back for the entry points that read bit planes (the reference's PackedMatrix.planes,
 * bitplane.py:79-122; batch_distances, distance.py:44-62; the index files, index.py:191-255).  Padding documents come back as
 * zeros, as the quantizer writes them. */
int xfbq_restore_codes_from_nibbles(const void *nibbles_dev, int64_t n, int64_t dim, int width, void *db_out_dev, void *stream);
int xfbq_restore_codes_from_tiles(const void *tiles_dev, int64_t n, int64_t dim, int width, void *db_out_dev, void *stream);
/* Which layout the preferred plan of a scan reads: XFBQ_LAYOUT_TILES (tcgen05 engine), XFBQ_LAYOUT_NIBBLES (mma.sync engine /
 * single-launch search) or 0 (XOR/POPC kernels on the bit planes). */
int xfbq_scan_layouts(int64_t n, int64_t dim, int doc_bits, int64_t nq, int query_bits, int k);
/* Both in one buffer, [nibble layout][byte tiles] (ABI revision 1): */
int64_t xfbq_derived_bytes(int64_t n, int64_t dim, int width);  /* width > 4: byte tiles only (no nibble region) */
int xfbq_build_derived(const void *db_dev, int64_t n, int64_t dim, int width, void *derived_out_dev, void *stream);
/* the same for width <= 4 (kept for callers of ABI revision 1) */
int64_t xfbq_nibble_bytes(int64_t n, int64_t dim);
int xfbq_planes_to_nibbles(const void *db_dev, int64_t n, int64_t dim, int width, void *nibbles_out_dev,
                           void *stream);

/*
 * batch_distances (distance.py:44-62 -> _kernels.py:56-69): distances from one
 * packed query (query layout, nq = 1) to every document; out_dev is uint64[n].
 */
int xfbq_batch_distances(const void *db_dev, int64_t n, int64_t dim, int doc_bits,
                         const uint32_t *q_dev, int query_bits, uint64_t *out_dev, void *stream);

/*
 * Candidate gather of k_select (search.py:206-216 after the histogram threshold, _kernels.py:56-69 for the
 * distances): one pass over the codes for one packed query, no distance array.  *count_out_dev (device
 * uint64, zeroed by the call) receives the number of documents with distance <= threshold; when
 * ids_out_dev is not NULL the first min(count, cap) of their row ids are written to it in no particular
 * order (the caller sorts: search.py:129-131).  count > cap means the id list is incomplete.
 */
int xfbq_collect_candidates(const void *db_dev, int64_t n, int64_t dim, int doc_bits, const uint32_t *q_dev,
                            int query_bits, int64_t threshold, int64_t *ids_out_dev, int64_t cap,
                            uint64_t *count_out_dev, void *stream);

/*
 * estimate_scale (index.py:123-138: 1 / np.quantile(|x|, p)).  numpy's "linear" quantile interpolates between two
 * order statistics of the flattened array; this call finds them exactly: out2_dev[0] / out2_dev[1] receive the
 * rank_lo-th and rank_hi-th smallest |x| (0-based ranks over the `count` contiguous elements at x_dev;
 * 0 <= rank_lo <= rank_hi < count), *nan_count_dev the number of NaN entries (they take no rank: numpy returns NaN
 * when there is one).  Most-significant-digit radix select on the float bit patterns, 11 bits per pass.
 * workspace_dev: xfbq_select_workspace_bytes() bytes, 8-byte aligned.
 */
int64_t xfbq_select_workspace_bytes(void);
int xfbq_abs_order_stats_f32(const float *x_dev, int64_t count, int64_t rank_lo, int64_t rank_hi, void *workspace_dev,
                             int64_t workspace_bytes, float *out2_dev, uint64_t *nan_count_dev, void *stream);
int xfbq_abs_order_stats_f64(const double *x_dev, int64_t count, int64_t rank_lo, int64_t rank_hi, void *workspace_dev,
                             int64_t workspace_bytes, double *out2_dev, uint64_t *nan_count_dev, void *stream);

/*
 * Float re-rank of k_select's candidates (refine, search.py:153-157 + _rank_hits :129-131; originals widened to
 * float64 as index.py:106-120): sims[c] = sum_k double(rows[r_c][k]) * q_dev[k] accumulated in float64, then the k
 * best (similarity desc, id asc) to sims_out_dev[k] / ids_out_dev[k] (slots beyond `count` hold 0.0 / -1).
 * r_c = ids_dev[c], or c when rows_gathered != 0 (rows_dev then holds the candidates' rows in candidate order and n
 * is ignored).  ids_dev[c] are the row ids reported and used as tie-break.  1 <= k <= XFBQ_MAX_K.
 */
int64_t xfbq_refine_workspace_bytes(int64_t count, int k);
int xfbq_refine_f32(const float *rows_dev, int64_t n, int64_t dim, int64_t ld, int rows_gathered, const int64_t *ids_dev,
                    int64_t count, const double *q_dev, int k, double *sims_out_dev, int64_t *ids_out_dev,
                    void *workspace_dev, int64_t workspace_bytes, void *stream);

/* The same gather from the nibble layout (doc_bits <= 4, query_bits <= 7, dim <= 512): the exact integer form of the distance on
 * dp4a, HBM-bound instead of POPC-bound; identical counts and ids. */
int xfbq_collect_candidates_nibbles(const void *nibbles_dev, int64_t n, int64_t dim, int doc_bits, const uint32_t *q_dev,
                                    int query_bits, int64_t threshold, int64_t *ids_out_dev, int64_t cap,
                                    uint64_t *count_out_dev, void *stream);

/*
 * The stand-alone histogram / gather stage of the reference (search.py:70-126), for callers that hold a distance array
 * (int64 on the device): DistanceHistogram.from_distances = xfbq_distance_histogram (*out_of_range_dev counts values outside
 * [0, bins)), kth_smallest = xfbq_histogram_kth (smallest t with >= k distances <= t), gather_candidates = xfbq_gather_le_count
 * (the number of rows with d <= threshold lands in workspace word [ceil(n / 65536)]) + xfbq_gather_le_ids (their ids,
 * ascending).  k_select itself never materialises the array (xfbq_scan_topk + xfbq_collect_candidates).
 */
int xfbq_distance_histogram(const int64_t *dist_dev, int64_t n, int64_t bins, uint64_t *hist_dev, uint64_t *out_of_range_dev, void *stream);
int xfbq_histogram_kth(const uint64_t *hist_dev, int64_t bins, int64_t k, int64_t *kth_out_dev, void *stream);
int64_t xfbq_gather_workspace_bytes(int64_t n);
int xfbq_gather_le_count(const int64_t *dist_dev, int64_t n, int64_t threshold, void *workspace_dev, int64_t workspace_bytes, void *stream);
int xfbq_gather_le_ids(const int64_t *dist_dev, int64_t n, int64_t threshold, const void *workspace_dev, int64_t *ids_out_dev, void *stream);

/*
 * Fused scan + top-K: for each of nq queries the k smallest keys
 * (distance << 32 | row_offset + row) over the n documents, ascending, written
 * to keys_out_dev[nq][k] (slots beyond min(k, n) hold UINT64_MAX).  No score
 * matrix is materialised.  Replaces, per query, batch_distances + the
 * no-originals ranking of k_select (search.py:206-216, :159-172, :129-131).
 * workspace_dev must hold xfbq_scan_workspace_bytes(...) bytes.
 * 1 <= k <= XFBQ_MAX_K;  row_offset + n <= 2^32.
 * nibbles_dev: optional derived layouts of the codes (xfbq_planes_to_nibbles).
 * When given (query_bits <= 7, dim <= 1024, k <= 1024) the scan runs on the integer tensor path -- tcgen05.mma
 * kind::i8 with accumulators in tensor memory for >= 17 queries (any batch size when doc_bits > 4 or dim > 512),
 * mma.sync (IMMA) below (doc_bits <= 4, dim <= 512) -- with identical results; when NULL, or outside those
 * shapes, the XOR/POPC kernels scan the bit planes.  XFBQ_ENGINE=umma|imma|popc forces one engine.
 */
int64_t xfbq_scan_workspace_bytes(int64_t n, int64_t dim, int doc_bits, int64_t nq,
                                  int query_bits, int k, int have_nibbles);
/* Launch plan xfbq_scan_topk will use on the current device, for reporting:
 * plan_out[0] = queries per CTA tile, [1] = query tiles, [2] = document splits (partial results
 * merged afterwards), [3] = candidate-list capacity per query, [4] = engine: 3 tcgen05, 2 mma.sync,
 * 1 specialised POPC kernel, 0 generic POPC kernel, [5] = dynamic shared memory bytes per CTA. */
int xfbq_scan_plan(int64_t n, int64_t dim, int doc_bits, int64_t nq, int query_bits, int k,
                   int have_nibbles, int32_t plan_out[6]);
int xfbq_scan_topk(const void *db_dev, const void *nibbles_dev, int64_t n, int64_t dim, int doc_bits,
                   const uint32_t *q_dev, int64_t nq, int query_bits, int k, int64_t row_offset,
                   uint64_t *keys_out_dev, void *workspace_dev, int64_t workspace_bytes,
                   void *stream);
/* The same with the two derived layouts passed separately (either may be NULL; the `have_nibbles` argument of
 * xfbq_scan_workspace_bytes / xfbq_scan_plan is then XFBQ_LAYOUT_NIBBLES | XFBQ_LAYOUT_TILES as available; 1 = both).
 * `db_dev` may be NULL when xfbq_scan_layouts() names a derived layout for the shape and that layout is passed: only the XOR/POPC
 * kernels read the packed codes (see xfbq_restore_codes_from_*).  The same holds for xfbq_search_small_* / xfbq_kselect_small_f64. */
int xfbq_scan_topk_layouts(const void *db_dev, const void *nibbles_dev, const void *tiles_dev, int64_t n, int64_t dim, int doc_bits,
                           const uint32_t *q_dev, int64_t nq, int query_bits, int k, int64_t row_offset,
                           uint64_t *keys_out_dev, void *workspace_dev, int64_t workspace_bytes, void *stream);

/*
 * Single-launch search for small batches (1 <= nq <= 16, doc_bits <= 4, query_bits <= 7, dim <= 512, k <= 1024, databases of
 * a million rows and more): float queries in, keys out, ONE cooperative kernel -- the query quantizer (quantize_vector,
 * bitplane.py:214-222), query preparation, threshold seeding, the HBM-bound scan and the merge (k_select's no-originals
 * ranking, search.py:159-172, :129-131) with grid-wide barriers in between, instead of ten launches.
 * xfbq_search_small_workspace_bytes returns 0 for shapes it does not take (use xfbq_quantize_queries_* + xfbq_scan_topk).
 * *nonfinite_dev (device uint64, NOT zeroed by the call) += the non-finite scaled query values found; a query holding one is
 * answered with empty keys (UINT64_MAX) -- the reference raises InvalidInputError (quant.py:142-143), which the caller does
 * when it reads the counter.  nibbles_dev: xfbq_build_derived / xfbq_planes_to_nibbles output.  Results are identical to
 * xfbq_scan_topk on the quantized queries.
 */
int64_t xfbq_search_small_workspace_bytes(int64_t n, int64_t dim, int doc_bits, int64_t nq, int query_bits, int k);
int xfbq_search_small_f32(const void *db_dev, const void *nibbles_dev, int64_t n, int64_t dim, int doc_bits, const float *queries_dev,
                          int64_t nq, int64_t ld, double scale, int query_bits, int k, int64_t row_offset, uint64_t *keys_out_dev,
                          uint64_t *nonfinite_dev, void *workspace_dev, int64_t workspace_bytes, void *stream);
int xfbq_search_small_f64(const void *db_dev, const void *nibbles_dev, int64_t n, int64_t dim, int doc_bits, const double *queries_dev,
                          int64_t nq, int64_t ld, double scale, int query_bits, int k, int64_t row_offset, uint64_t *keys_out_dev,
                          uint64_t *nonfinite_dev, void *workspace_dev, int64_t workspace_bytes, void *stream);

/*
 * k_select in one launch (search.py:188-232 up to the re-rank): the search above plus the histogram / gather stage -- per query
 * the number of rows with distance <= (k-th distance + extra_distance) in cand_count_out_dev[nq] and, when cand_ids_out_dev is
 * not NULL, the first min(count, cand_cap) of their row ids (unordered) in cand_ids_out_dev[nq][cand_cap].  The scan keeps every
 * such row in its candidate lists unless a list overflowed and was cut: then *inexact_out_dev != 0 and the caller runs
 * xfbq_collect_candidates* instead (large extra_distance, heavy ties).  float64 queries (SearchRequest.query is float64).
 */
int xfbq_kselect_small_f64(const void *db_dev, const void *nibbles_dev, int64_t n, int64_t dim, int doc_bits, const double *queries_dev,
                           int64_t nq, int64_t ld, double scale, int query_bits, int k, int64_t extra_distance, int64_t row_offset,
                           uint64_t *keys_out_dev, uint64_t *cand_count_out_dev, int64_t *cand_ids_out_dev, int64_t cand_cap,
                           int *inexact_out_dev, uint64_t *nonfinite_dev, void *workspace_dev, int64_t workspace_bytes, void *stream);

/*
 * Merge `parts` partial results keys_in_dev[parts][nq][k] (each row ascending,
 * UINT64_MAX padded) into keys_out_dev[nq][k]: the exchange step after the
 * per-GPU scans (no reference code; semantics of search.py:129-131: total order
 * on (distance, id), so the result is independent of the partition).
 */
int xfbq_merge_topk(const uint64_t *keys_in_dev, int parts, int64_t nq, int k,
                    uint64_t *keys_out_dev, void *stream);

/* Split keys into int64 distances and int64 row ids (-1 / -1 for empty slots). */
int xfbq_unpack_keys(const uint64_t *keys_dev, int64_t count, int64_t *dist_out_dev,
                     int64_t *id_out_dev, void *stream);

/* Measurement aid: when enabled, the calling host thread records CUDA events on the scan's stream
 * around the dominant kernel of every xfbq_scan_topk call (the scan itself, not query preparation
 * or the merge); xfbq_last_scan_ms synchronises on the last one and returns its duration. */
int xfbq_set_timing(int enable);
int xfbq_last_scan_ms(float *ms_out);
/* Mean duration of the dominant kernel over the timed launches since xfbq_set_timing(1) (the last 64 are kept). */
int xfbq_scan_ms_mean(float *mean_ms_out, int *launches_out);
/* Debug hook (per host thread): device buffer of gridDim.x * 12 uint64 counters that the tcgen05 scan
 * kernel of the following xfbq_scan_topk calls fills with cycles spent waiting per role
 * (tools/umma_profile.py); NULL switches it off. */
int xfbq_debug_profile(void *device_counters);

/* Number of kernels this library has launched in the calling process (for bench accounting). */
int64_t xfbq_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* XFBQ_B200_H */
