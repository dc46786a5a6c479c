/*
 * xfbq_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This file is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2008_02002_b200/) must never import, link or call anything here.
 *
 * Parity is PINNED: oracle/gen_golden.py runs the unmodified reference package
 * (/root/reference/pkg/src/xfbq) in the build container and commits its outputs
 * under tests/golden/; tests/test_oracle_golden.py checks every function below
 * against those fixtures and against the reference's own worked examples.
 *
 * Each function cites the reference file:line it restates.  Loop orders follow
 * the reference so the timing of the "port" baseline is representative.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define XO_EXPORT __attribute__((visibility("default")))

/* bitplane.py:29-30  words_needed(dim) = ceil(dim / 64) */
XO_EXPORT int64_t xo_words_needed(int64_t dim) { return (dim + 63) / 64; }

/* distance.py:25-29 + quant.py:113-115  dim * (2^wx - 1) * (2^wy - 1) */
XO_EXPORT int64_t xo_distance_upper_bound(int64_t dim, int wx, int wy) {
    return dim * (int64_t)((1 << wx) - 1) * (int64_t)((1 << wy) - 1);
}

/*
 * quant.py:138-148  quantize_values
 *   odd  = 2*floor(x * 2^(w-1)) + 1 ; clip(odd, -hi, hi) ; code = (hi - odd) * 0.5
 * Returns the number of non-finite inputs (the reference raises InvalidInputError
 * when that is non-zero, quant.py:142-143); codes for those entries are undefined.
 */
XO_EXPORT int64_t xo_quantize_values(const double *x, int64_t m, int width, uint8_t *codes) {
    const double hi = (double)((1 << width) - 1);
    const double half_range = (double)(1 << (width - 1));
    int64_t bad = 0;
    for (int64_t t = 0; t < m; ++t) {
        double v = x[t];
        if (!isfinite(v)) { ++bad; codes[t] = 0; continue; }
        double odd = 2.0 * floor(v * half_range) + 1.0;
        if (odd < -hi) odd = -hi;
        if (odd > hi) odd = hi;
        codes[t] = (uint8_t)((hi - odd) * 0.5);
    }
    return bad;
}

/*
 * bitplane.py:151-163  _pack_code_matrix: (n, dim) u8 codes -> (width, words, n) u64.
 * Plane b, word k/64, bit k%64 (little-endian bit numbering) holds bit b of
 * codes[r, k]; padding bits stay zero.
 */
XO_EXPORT void xo_pack_code_matrix(const uint8_t *codes, int64_t n, int64_t dim, int width,
                                   uint64_t *planes) {
    const int64_t nwords = xo_words_needed(dim);
    memset(planes, 0, (size_t)width * (size_t)nwords * (size_t)n * sizeof(uint64_t));
    for (int b = 0; b < width; ++b)
        for (int64_t r = 0; r < n; ++r)
            for (int64_t k = 0; k < dim; ++k) {
                uint64_t bit = (uint64_t)((codes[r * dim + k] >> b) & 1u);
                planes[((int64_t)b * nwords + k / 64) * n + r] |= bit << (k % 64);
            }
}

/*
 * bitplane.py:225-233 quantize_matrix on float32 input as build_index feeds it
 * (index.py:155 casts to float32, bitplane.py:229 widens to float64, :232 scales).
 * Row-chunked so the temporaries stay small; returns the non-finite count of the
 * SCALED values (quant.py:142).
 */
XO_EXPORT int64_t xo_quantize_matrix_f32(const float *x, int64_t n, int64_t dim, int64_t ld,
                                         double scale, int width, uint64_t *planes) {
    const int64_t nwords = xo_words_needed(dim);
    const double hi = (double)((1 << width) - 1);
    const double half_range = (double)(1 << (width - 1));
    int64_t bad = 0;
    memset(planes, 0, (size_t)width * (size_t)nwords * (size_t)n * sizeof(uint64_t));
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t k = 0; k < dim; ++k) {
            double v = (double)x[r * ld + k] * scale; /* bitplane.py:232 */
            if (!isfinite(v)) { ++bad; continue; }
            double odd = 2.0 * floor(v * half_range) + 1.0; /* quant.py:146 */
            if (odd < -hi) odd = -hi;
            if (odd > hi) odd = hi;
            unsigned code = (unsigned)((hi - odd) * 0.5);
            for (int b = 0; b < width; ++b)
                planes[((int64_t)b * nwords + k / 64) * n + r] |=
                    (uint64_t)((code >> b) & 1u) << (k % 64);
        }
    }
    return bad;
}

/* Same for float64 input (quantize_vector on a float64 query, bitplane.py:214-222). */
XO_EXPORT int64_t xo_quantize_matrix_f64(const double *x, int64_t n, int64_t dim, int64_t ld,
                                         double scale, int width, uint64_t *planes) {
    const int64_t nwords = xo_words_needed(dim);
    const double hi = (double)((1 << width) - 1);
    const double half_range = (double)(1 << (width - 1));
    int64_t bad = 0;
    memset(planes, 0, (size_t)width * (size_t)nwords * (size_t)n * sizeof(uint64_t));
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t k = 0; k < dim; ++k) {
            double v = x[r * ld + k] * scale;
            if (!isfinite(v)) { ++bad; continue; }
            double odd = 2.0 * floor(v * half_range) + 1.0;
            if (odd < -hi) odd = -hi;
            if (odd > hi) odd = hi;
            unsigned code = (unsigned)((hi - odd) * 0.5);
            for (int b = 0; b < width; ++b)
                planes[((int64_t)b * nwords + k / 64) * n + r] |=
                    (uint64_t)((code >> b) & 1u) << (k % 64);
        }
    }
    return bad;
}

/*
 * _kernels.py:56-69  _batch_distances_jit.  Same pass structure: plane pair (i, j)
 * outermost, then word, documents innermost with a read-modify-write of out[k].
 *   out[k] = sum_{i<wd} sum_{j<wq} sum_w popcount(D[i,w,k] ^ Q[j,w]) << (i+j)
 */
XO_EXPORT void xo_batch_distances(const uint64_t *doc_planes, int wd, int64_t nwords, int64_t n,
                                  const uint64_t *query_planes, int wq, uint64_t *out) {
    for (int64_t k = 0; k < n; ++k) out[k] = 0;
    for (int i = 0; i < wd; ++i)
        for (int j = 0; j < wq; ++j) {
            const int shift = i + j;
            for (int64_t w = 0; w < nwords; ++w) {
                const uint64_t *words = doc_planes + ((int64_t)i * nwords + w) * n;
                const uint64_t qword = query_planes[(int64_t)j * nwords + w];
                for (int64_t k = 0; k < n; ++k)
                    out[k] += (uint64_t)__builtin_popcountll(words[k] ^ qword) << shift;
            }
        }
}

/* distance.py:32-41  packed_distance (pairwise definition twin). */
XO_EXPORT uint64_t xo_packed_distance(const uint64_t *x, int wx, const uint64_t *y, int wy,
                                      int64_t nwords) {
    uint64_t total = 0;
    for (int i = 0; i < wx; ++i)
        for (int j = 0; j < wy; ++j) {
            uint64_t pc = 0;
            for (int64_t w = 0; w < nwords; ++w)
                pc += (uint64_t)__builtin_popcountll(x[i * nwords + w] ^ y[j * nwords + w]);
            total += pc << (i + j);
        }
    return total;
}

typedef struct { uint64_t d; int64_t id; } xo_pair;

static int xo_pair_cmp(const void *a, const void *b) {
    const xo_pair *p = (const xo_pair *)a, *q = (const xo_pair *)b;
    if (p->d != q->d) return p->d < q->d ? -1 : 1;
    if (p->id != q->id) return p->id < q->id ? -1 : 1;
    return 0;
}

/*
 * search.py:129-131 _rank_hits on the no-originals branch (search.py:159-172):
 * similarity is a strictly decreasing affine map of the distance, so
 * lexsort((ids, -sims))[:k] == order by (distance asc, id asc).  SURVEY 8c:
 *   order = np.lexsort((np.arange(n), d))[:min(k, n)]
 * Threshold pre-filter keeps it O(n + m log m); the result is the exact sort.
 * Returns the number of hits written (min(k, n)).
 */
XO_EXPORT int64_t xo_topk(const uint64_t *dists, int64_t n, int64_t k, uint64_t *out_d,
                          int64_t *out_id) {
    if (k > n) k = n;
    if (k <= 0) return 0;
    /* kth smallest distance by counting (search.py:101-117 histogram idea) */
    uint64_t dmax = 0;
    for (int64_t t = 0; t < n; ++t) if (dists[t] > dmax) dmax = dists[t];
    xo_pair *cand = NULL;
    int64_t m = 0;
    if (dmax < (1u << 22)) {
        int64_t *bins = (int64_t *)calloc((size_t)dmax + 1, sizeof(int64_t));
        for (int64_t t = 0; t < n; ++t) bins[dists[t]]++;
        uint64_t thr = 0; int64_t cum = 0;
        for (uint64_t v = 0; v <= dmax; ++v) { cum += bins[v]; if (cum >= k) { thr = v; break; } }
        free(bins);
        for (int64_t t = 0; t < n; ++t) if (dists[t] <= thr) ++m;
        cand = (xo_pair *)malloc((size_t)m * sizeof(xo_pair));
        m = 0;
        for (int64_t t = 0; t < n; ++t)
            if (dists[t] <= thr) { cand[m].d = dists[t]; cand[m].id = t; ++m; }
    } else {
        cand = (xo_pair *)malloc((size_t)n * sizeof(xo_pair));
        for (int64_t t = 0; t < n; ++t) { cand[t].d = dists[t]; cand[t].id = t; }
        m = n;
    }
    qsort(cand, (size_t)m, sizeof(xo_pair), xo_pair_cmp);
    for (int64_t t = 0; t < k; ++t) { out_d[t] = cand[t].d; out_id[t] = cand[t].id; }
    free(cand);
    return k;
}

/*
 * Batched oracle (SURVEY 8c composition): per query, batch_distances then the
 * (dist asc, id asc) top-k.  Threads split the QUERIES, as the reference's own
 * bench does with its thread pool (bench.py:254-259); each query is the
 * single-threaded reference pass.  out_d/out_id are [nq, kk], kk = min(k, n).
 * row_offset is added to the ids (shard-local -> global row numbers).
 */
XO_EXPORT int64_t xo_search(const uint64_t *doc_planes, int wd, int64_t nwords, int64_t n,
                            const uint64_t *query_planes /* [nq, wq, nwords] */, int64_t nq,
                            int wq, int64_t k, int64_t row_offset, int threads,
                            uint64_t *out_d, int64_t *out_id) {
    const int64_t kk = k < n ? k : n;
    if (kk <= 0 || nq <= 0) return kk < 0 ? 0 : kk;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        uint64_t *scratch = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t q = 0; q < nq; ++q) {
            xo_batch_distances(doc_planes, wd, nwords, n,
                               query_planes + q * (int64_t)wq * nwords, wq, scratch);
            xo_topk(scratch, n, kk, out_d + q * kk, out_id + q * kk);
            for (int64_t t = 0; t < kk; ++t) out_id[q * kk + t] += row_offset;
        }
        free(scratch);
    }
    return kk;
}

XO_EXPORT int xo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
