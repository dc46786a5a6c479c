// xfbq_select.cuh -- exact order statistics of |x| (estimate_scale, index.py:123-138) and the float re-rank of
// k_select's candidates (search.py:153-157, index.py:106-120) -- included by xfbq_b200.cu.
//
// estimate_scale = 1 / np.quantile(|x|, p): numpy's "linear" method interpolates between TWO order statistics of
// the flattened array (ranks floor((n-1)p) and the next one).  The data-sized part -- finding those two values
// exactly -- is a most-significant-digit radix select on the bit patterns of |x| (non-negative IEEE floats order
// like unsigned integers), 11 bits per pass: a histogram pass over every element that still matches the prefix
// found so far, then a one-block pick of the digit that holds the rank.  Three passes for float32, six for
// float64; both ranks are tracked at once (they nearly always share every digit but the last).  The interpolation
// itself is a handful of scalar operations on the host (paper_2008_02002_b200/index.py restates numpy's).
#pragma once

namespace sel {

constexpr int DIGIT_BITS = 11;
constexpr int BINS = 1 << DIGIT_BITS;
constexpr int COPIES = 8;  // shared-memory histogram copies (lane & 7): unit-norm data puts most first digits in a few bins

struct State {              // device-resident, one per call (workspace)
    unsigned long long hist[2][BINS];
    unsigned long long prefix[2];   // digits found so far, right-aligned
    long long rank[2];              // rank still to find among the elements matching prefix[t]
    unsigned long long nan_count;
    int same;                       // both targets share prefix[0]: one histogram serves both
    int pad;
};

template <typename T> struct KeyOf;
template <> struct KeyOf<float> {
    typedef uint32_t type;
    static constexpr int BITS = 32;
    static __device__ __forceinline__ uint32_t key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }
    static __device__ __forceinline__ bool is_nan(uint32_t k) { return k > 0x7F800000u; }
};
template <> struct KeyOf<double> {
    typedef unsigned long long type;
    static constexpr int BITS = 64;
    static __device__ __forceinline__ unsigned long long key(double v) {
        return static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7FFFFFFFFFFFFFFFull;
    }
    static __device__ __forceinline__ bool is_nan(unsigned long long k) { return k > 0x7FF0000000000000ull; }
};

__global__ void init_state_kernel(State *st, long long rank_lo, long long rank_hi) {
    for (int i = threadIdx.x; i < 2 * BINS; i += blockDim.x) (&st->hist[0][0])[i] = 0ull;
    if (threadIdx.x == 0) {
        st->prefix[0] = st->prefix[1] = 0ull;
        st->rank[0] = rank_lo; st->rank[1] = rank_hi;
        st->nan_count = 0ull; st->same = 1; st->pad = 0;
    }
}

// Histogram of digit [lo_bit, lo_bit + nbits) over the elements whose higher bits equal the prefix of a target.
// FIRST: no prefix yet (every element counts; NaNs are counted on the side -- numpy's quantile returns NaN then).
template <typename T, bool FIRST>
__global__ void __launch_bounds__(256) hist_kernel(const T *__restrict__ x, int64_t count, int lo_bit, int nbits, State *st) {
    typedef typename KeyOf<T>::type K;
    extern __shared__ uint32_t sh[];  // [COPIES][BINS]
    for (int i = threadIdx.x; i < COPIES * BINS; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    const int same = FIRST ? 1 : st->same;
    const K p0 = static_cast<K>(st->prefix[0]), p1 = static_cast<K>(st->prefix[1]);
    const int hi_bit = lo_bit + nbits;
    const uint32_t mask = (1u << nbits) - 1u;
    const int lane = threadIdx.x & 31;
    // same prefix: 8 copies by lane; different prefixes: target t owns copies 4t .. 4t + 3
    uint32_t *h0 = sh + (same ? (lane & 7) : (lane & 3)) * BINS;
    uint32_t *h1 = sh + (4 + (lane & 3)) * BINS;
    unsigned long long nans = 0;
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte load
    const int64_t nvec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) ? count / V : 0;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    // FIRST pass: every element counts and most of them share a few digits (the exponent of unit-norm components), so the
    // lanes of a warp that hold the same digit are found with match.any and ONE of them adds their number: one shared-memory
    // atomic per distinct digit and warp instruction instead of 32 colliding ones (103 -> see profiles for 1G values).
    // Later passes count only the elements under the prefix (one in 2 048 or fewer): plain atomics.
    auto visit_first = [&](T v, bool valid) {   // warp-uniform call: every lane takes part in the vote
        const K k = KeyOf<T>::key(v);
        const bool nan = valid && KeyOf<T>::is_nan(k);
        if (nan) ++nans;
        const uint32_t d = (valid && !nan) ? (static_cast<uint32_t>(k >> lo_bit) & mask) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&h0[d], static_cast<uint32_t>(__popc(peers)));
    };
    auto visit = [&](T v) {
        const K k = KeyOf<T>::key(v);
        const K hi = hi_bit >= KeyOf<T>::BITS ? static_cast<K>(0) : static_cast<K>(k >> hi_bit);
        const uint32_t d = static_cast<uint32_t>(k >> lo_bit) & mask;
        if (hi == p0) atomicAdd(&h0[d], 1u);
        if (!same && hi == p1) atomicAdd(&h1[d], 1u);
    };
    const uint4 *xv = reinterpret_cast<const uint4 *>(x);
    if (FIRST) {
        const int64_t nvec_round = (nvec + 31) & ~static_cast<int64_t>(31);  // whole warps stay in the loop for the vote
        for (int64_t i = tid; i < nvec_round; i += nthreads) {
            const bool in = i < nvec;
            const uint4 w = in ? __ldg(xv + i) : make_uint4(0u, 0u, 0u, 0u);
            T e[V];
            memcpy(e, &w, 16);
#pragma unroll
            for (int j = 0; j < V; ++j) visit_first(e[j], in);
        }
        const int64_t tail0 = nvec * V, tail_round = (count - tail0 + 31) & ~static_cast<int64_t>(31);
        for (int64_t i = tid; i < tail_round; i += nthreads) {
            const bool in = tail0 + i < count;
            visit_first(in ? x[tail0 + i] : static_cast<T>(0), in);
        }
    } else {
#pragma unroll 2
        for (int64_t i = tid; i < nvec; i += nthreads) {
            const uint4 w = __ldg(xv + i);
            T e[V];
            memcpy(e, &w, 16);
#pragma unroll
            for (int j = 0; j < V; ++j) visit(e[j]);
        }
        for (int64_t i = nvec * V + tid; i < count; i += nthreads) visit(x[i]);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < BINS; b += blockDim.x) {
        uint32_t c0 = 0, c1 = 0;
        if (same) {
#pragma unroll
            for (int c = 0; c < COPIES; ++c) c0 += sh[c * BINS + b];
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) { c0 += sh[c * BINS + b]; c1 += sh[(4 + c) * BINS + b]; }
        }
        if (c0) atomicAdd(&st->hist[0][b], static_cast<unsigned long long>(c0));
        if (c1) atomicAdd(&st->hist[1][b], static_cast<unsigned long long>(c1));
    }
    if (FIRST) {
#pragma unroll
        for (int o = 16; o; o >>= 1) nans += __shfl_xor_sync(0xffffffffu, nans, o);
        if (lane == 0 && nans) atomicAdd(&st->nan_count, nans);
    }
}

// One block: for each target, the digit whose bin holds the rank; prefix and rank move on, histograms are cleared.
__global__ void __launch_bounds__(1024) pick_kernel(State *st, int nbits) {
    __shared__ int s_digit[2];
    __shared__ long long s_below[2];
    const int same = st->same;
    for (int t = 0; t < 2; ++t) {
        const unsigned long long *h = st->hist[same ? 0 : t];
        const long long want = st->rank[t];
        // inclusive prefix sums of the bins (2048 bins, 1024 threads: two bins per thread, block scan)
        const int b0 = 2 * threadIdx.x;
        const unsigned long long a = h[b0], b = h[b0 + 1];
        unsigned long long sum = a + b;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        unsigned long long inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        __shared__ unsigned long long s_warp[32];
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = s_warp[lane], wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long v = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += v;
            }
            s_warp[lane] = wi - w;  // exclusive
        }
        __syncthreads();
        const unsigned long long exc = s_warp[warp] + inc - sum;  // elements in bins below b0
        // the digit: smallest bin with inclusive count > want
        const unsigned long long w = static_cast<unsigned long long>(want);
        if (exc <= w && w < exc + a) { s_digit[t] = b0; s_below[t] = static_cast<long long>(exc); }
        else if (exc + a <= w && w < exc + a + b) { s_digit[t] = b0 + 1; s_below[t] = static_cast<long long>(exc + a); }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int t = 0; t < 2; ++t) {
            st->prefix[t] = (st->prefix[t] << nbits) | static_cast<unsigned long long>(s_digit[t]);
            st->rank[t] -= s_below[t];
        }
        st->same = st->prefix[0] == st->prefix[1];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * BINS; i += blockDim.x) (&st->hist[0][0])[i] = 0ull;
}

template <typename T>
__global__ void finish_kernel(const State *st, T *out2, unsigned long long *nan_out) {
    typedef typename KeyOf<T>::type K;
    if (threadIdx.x < 2) {
        const K k = static_cast<K>(st->prefix[threadIdx.x]);
        T v;
        memcpy(&v, &k, sizeof(T));
        out2[threadIdx.x] = v;
    }
    if (threadIdx.x == 0) *nan_out = st->nan_count;
}

// ------------------------------------------------------------------------------ float re-rank (search.py:153-157)
// sims[c] = sum_k double(rows[ids[c]][k]) * q[k], accumulated in float64 IN DIMENSION ORDER by pairwise halves the way
// a BLAS dot would not promise -- the reference's `rows @ q` goes through numpy's float64 matmul (pairwise / SIMD
// order unspecified), so the comparison with it is to 1e-12 relative, not bit-exact (tests state the tolerance).
// One warp per candidate: lanes stride the row (coalesced float32 loads), butterfly reduction.
template <typename T>
__global__ void __launch_bounds__(256) gather_dot_kernel(const T *__restrict__ rows, int64_t ld, int dim, const int64_t *__restrict__ ids,
                                                         int64_t count, const double *__restrict__ q, double *__restrict__ sims) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (c >= count) return;
    const T *row = rows + (ids ? ids[c] : c) * ld;  // ids == nullptr: the rows were gathered by the caller
    double acc = 0.0;
    for (int k = lane; k < dim; k += 32) acc = fma(static_cast<double>(row[k]), __ldg(q + k), acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sims[c] = acc;
}

// Rank keys of the re-rank: (similarity desc, id asc) == ascending (monotone key of -sim, id).  The float64 similarity
// maps to a uint64 whose unsigned order is the numeric order of -sim (search.py:129-131 lexsort((ids, -sims))).
__device__ __forceinline__ unsigned long long order_key_desc(double sim) {
    const double neg = 0.0 - sim;  // -0.0 and 0.0 rank equal, like numpy's comparison
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(neg));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double sim_of_key(unsigned long long key) {
    const unsigned long long b = (key & 0x8000000000000000ull) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
    return 0.0 - __longlong_as_double(static_cast<long long>(b));
}

struct RankPair { unsigned long long key; long long id; };
constexpr long long RANK_EMPTY = 0x7FFFFFFFFFFFFFFFll;
__device__ __forceinline__ bool pair_less(const RankPair &a, const RankPair &b) {
    return a.key < b.key || (a.key == b.key && a.id < b.id);
}

// Block-wide bounded top-k over a stream of pairs: buf[0, K2) holds the best so far (sorted after every flush),
// buf[K2, 2 K2) collects the pairs that beat the current k-th; a full upper half is folded in by one bitonic sort of
// the 2 K2 entries.  K2 = power of two >= max(k, blockDim.x).  Every thread of the block calls it with the same arguments.
template <typename Fetch>
__device__ void bounded_topk(RankPair *buf, int K2, int k, int64_t begin, int64_t end, Fetch fetch) {
    __shared__ int s_cnt;
    const RankPair inf{~0ull, RANK_EMPTY};
    for (int t = threadIdx.x; t < 2 * K2; t += blockDim.x) buf[t] = inf;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    auto fold = [&]() {  // sort buf[0, 2 K2): the K2 best end up in the lower half; ends on a barrier
        const int P = 2 * K2;
        for (int size = 2; size <= P; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                    const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const RankPair a = buf[lo], b = buf[hi];
                    if (pair_less(b, a) == up) { buf[lo] = b; buf[hi] = a; }
                }
                __syncthreads();
            }
        for (int t = threadIdx.x; t < K2; t += blockDim.x) buf[K2 + t] = inf;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
    };
    for (int64_t e0 = begin; e0 < end; e0 += blockDim.x) {
        const int c = s_cnt;
        __syncthreads();  // everyone has read the count: the branch is block-uniform
        if (c + static_cast<int>(blockDim.x) > K2) fold();
        const RankPair kth = buf[k - 1];  // inf until k pairs have been folded in
        const int64_t e = e0 + threadIdx.x;
        RankPair mine = inf;
        if (e < end) mine = fetch(e);
        const bool keep = mine.id != RANK_EMPTY && pair_less(mine, kth);
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        const int lane = threadIdx.x & 31;
        if (lane == 0 && m) base = atomicAdd(&s_cnt, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) buf[K2 + base + __popc(m & ((1u << lane) - 1u))] = mine;
        __syncthreads();
    }
    fold();
}

// Stage 1: block b ranks its contiguous share of the candidates and writes its k best pairs (RANK_EMPTY padded).
__global__ void __launch_bounds__(256) rank_partial_kernel(const double *__restrict__ sims, const int64_t *__restrict__ ids, int64_t count,
                                                          int k, int K2, RankPair *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char raw[];
    RankPair *buf = reinterpret_cast<RankPair *>(raw);
    const int64_t per = (count + gridDim.x - 1) / gridDim.x;
    const int64_t begin = static_cast<int64_t>(blockIdx.x) * per, end = min(count, begin + per);
    bounded_topk(buf, K2, k, begin, end, [&](int64_t e) { return RankPair{order_key_desc(sims[e]), ids[e]}; });
    for (int t = threadIdx.x; t < k; t += blockDim.x) part[static_cast<int64_t>(blockIdx.x) * k + t] = buf[t];
}

// Stage 2: one block ranks the partial results; hits leave as (id, float64 similarity), best first.
__global__ void __launch_bounds__(256) rank_final_kernel(const RankPair *__restrict__ part, int64_t count, int k, int K2,
                                                        double *__restrict__ out_sims, int64_t *__restrict__ out_ids) {
    extern __shared__ __align__(16) unsigned char raw[];
    RankPair *buf = reinterpret_cast<RankPair *>(raw);
    bounded_topk(buf, K2, k, 0, count, [&](int64_t e) { return part[e]; });
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        const bool real = buf[t].id != RANK_EMPTY;
        out_sims[t] = real ? sim_of_key(buf[t].key) : 0.0;
        out_ids[t] = real ? buf[t].id : -1;
    }
}


// ------------------------------------------------------------------------------ stand-alone histogram / gather
// histogram_kth_distance and gather_candidates of the reference (search.py:70-126) take a DISTANCE ARRAY; k_select here
// never materialises one (the fused scan's k-th key is the threshold), these kernels serve the stand-alone functions.
__global__ void __launch_bounds__(256) dist_histogram_kernel(const int64_t *__restrict__ d, int64_t n, int64_t bins,
                                                             unsigned long long *__restrict__ hist, unsigned long long *__restrict__ over) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    unsigned long long bad = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t v = d[i];
        if (v < 0 || v >= bins) ++bad; else atomicAdd(hist + v, 1ull);
    }
    if (bad) atomicAdd(over, bad);
}

// One block: smallest value t with at least k distances <= t (search.py:92-98: searchsorted(cumsum(bins), k, 'left')).
__global__ void __launch_bounds__(1024) hist_kth_kernel(const unsigned long long *__restrict__ hist, int64_t bins, unsigned long long k,
                                                        long long *__restrict__ out) {
    __shared__ unsigned long long s_part[1024];
    const int64_t per = (bins + blockDim.x - 1) / blockDim.x;
    const int64_t lo = threadIdx.x * per, hi = min(bins, lo + per);
    unsigned long long sum = 0;
    for (int64_t b = lo; b < hi; ++b) sum += hist[b];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        long long ans = bins;  // k > total: past the last bin (the caller clamps k to the total first)
        for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
            if (run + s_part[t] >= k) {
                for (int64_t b = t * per; b < min(bins, (t + 1) * per); ++b) {
                    run += hist[b];
                    if (run >= k) { ans = b; break; }
                }
                break;
            }
            run += s_part[t];
        }
        *out = ans;
    }
}

// ids with d <= threshold in ascending id order: per-block counts, then (after a host-side / device prefix) ordered writes.
__global__ void __launch_bounds__(256) count_le_kernel(const int64_t *__restrict__ d, int64_t n, int64_t thr, int64_t per_block,
                                                       unsigned long long *__restrict__ block_counts) {
    __shared__ unsigned long long s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * per_block, hi = min(n, lo + per_block);
    unsigned long long c = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) c += d[i] <= thr ? 1 : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s, c);
    __syncthreads();
    if (threadIdx.x == 0) block_counts[blockIdx.x] = s;
}
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(unsigned long long *__restrict__ v, int n) {  // one block, in place; v[n] = total
    __shared__ unsigned long long s_part[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(n, lo + per);
    unsigned long long sum = 0;
    for (int i = lo; i < hi; ++i) sum += v[i];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int t = 0; t < static_cast<int>(blockDim.x); ++t) { const unsigned long long c = s_part[t]; s_part[t] = run; run += c; }
        v[n] = run;
    }
    __syncthreads();
    unsigned long long run = s_part[threadIdx.x];
    for (int i = lo; i < hi; ++i) { const unsigned long long c = v[i]; v[i] = run; run += c; }
}
__global__ void __launch_bounds__(256) gather_le_kernel(const int64_t *__restrict__ d, int64_t n, int64_t thr, int64_t per_block,
                                                        const unsigned long long *__restrict__ block_offsets, int64_t *__restrict__ ids) {
    __shared__ unsigned long long s_base;
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * per_block, hi = min(n, lo + per_block);
    if (threadIdx.x == 0) s_base = block_offsets[blockIdx.x];
    __shared__ int s_warp[8];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t i0 = lo; i0 < hi; i0 += blockDim.x) {   // block-ordered compaction, 256 rows per round
        const int64_t i = i0 + threadIdx.x;
        const bool hit = i < hi && d[i] <= thr;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_warp[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < 8; ++w) { if (w < warp) before += s_warp[w]; total += s_warp[w]; }
        if (hit) ids[s_base + before + __popc(m & ((1u << lane) - 1u))] = i;
        __syncthreads();
        if (threadIdx.x == 0) s_base += total;
        __syncthreads();
    }
}


// ------------------------------------------------------------------------------ candidate gather on the nibble layout
// The gather stage of k_select (d <= threshold, search.py:120-126) from the row-major 4-bit copy of the codes with the exact
// integer form d = Dq - sum_k x_k (2 y_k - Aq) on dp4a: HBM-bound (0.2 ms per pass over 10M x 256), where the XOR/POPC form
// on the bit planes is POPC-bound (0.36 ms).  One thread per document; the query's s8 weights sit in shared memory in the
// order the nibble split produces: for group g of 32 dims and nibble word e, word 2e holds dims 32g + 8j + e (j = 0..3),
// word 2e + 1 dims 32g + 8j + 4 + e.
template <int C>
__global__ void __launch_bounds__(256)
collect_candidates_nib_kernel(const uint4 *__restrict__ nib, int64_t n, int dim, int wd, const uint32_t *__restrict__ q, int wq,
                              uint32_t threshold, int64_t *__restrict__ ids_out, int64_t cap, unsigned long long *__restrict__ counts) {
    __shared__ __align__(16) uint32_t s_w[32 * C];
    __shared__ int s_dq;
    const int W = 4 * C;
    const int Aq = (1 << wq) - 1, Ad = (1 << wd) - 1;
    if (threadIdx.x == 0) s_dq = 0;
    __syncthreads();
    int sy = 0;
    for (int ow = threadIdx.x; ow < 32 * C; ow += blockDim.x) {
        const int g = ow >> 3, e = (ow >> 1) & 3, hi = ow & 1;
        uint32_t packed = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int d = 32 * g + 8 * j + 4 * hi + e;
            if (d < dim) {
                int y = 0;
                for (int jq = 0; jq < wq; ++jq) y |= static_cast<int>((q[jq * W + (d >> 5)] >> (d & 31)) & 1u) << jq;
                sy += y;
                packed |= (static_cast<uint32_t>(2 * y - Aq) & 0xFFu) << (8 * j);
            }
        }
        s_w[ow] = packed;
    }
    if (sy) atomicAdd(&s_dq, Ad * sy);
    __syncthreads();
    const int dq = s_dq;
    const int lane = threadIdx.x & 31;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n_round = (n + 31) & ~static_cast<int64_t>(31);  // whole warps stay in the loop for the vote
    for (int64_t doc = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; doc < n_round; doc += stride) {
        int acc = 0;
        if (doc < n) {
            const uint4 *row = nib + doc * W;
#pragma unroll
            for (int g = 0; g < W; ++g) {
                const uint4 v = __ldg(row + g);
                const uint4 w0 = *reinterpret_cast<const uint4 *>(s_w + 8 * g), w1 = *reinterpret_cast<const uint4 *>(s_w + 8 * g + 4);
                acc = umma::dp4a_su(w0.x, v.x & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w0.y, (v.x >> 4) & 0x0F0F0F0Fu, acc);
                acc = umma::dp4a_su(w0.z, v.y & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w0.w, (v.y >> 4) & 0x0F0F0F0Fu, acc);
                acc = umma::dp4a_su(w1.x, v.z & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w1.y, (v.z >> 4) & 0x0F0F0F0Fu, acc);
                acc = umma::dp4a_su(w1.z, v.w & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w1.w, (v.w >> 4) & 0x0F0F0F0Fu, acc);
            }
        }
        const bool hit = doc < n && static_cast<uint32_t>(dq - acc) <= threshold;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (m) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(counts, static_cast<unsigned long long>(__popc(m)));
            base = __shfl_sync(0xffffffffu, base, 0);
            const int64_t pos = static_cast<int64_t>(base) + __popc(m & ((1u << lane) - 1u));
            if (hit && ids_out && pos < cap) ids_out[pos] = doc;
        }
    }
}


// The same for row lengths that divide a warp's 512-byte load (C = 1, 2, 4: W = 4, 8, 16 uint4 per document): a warp reads the
// rows of 32 consecutive documents as 32 W / 32 fully coalesced 512-byte loads; lane l always meets group l % W, so its eight
// weight words live in registers, and the W lanes of a document add their partial dot products with log2(W) shuffles.
template <int C>
__global__ void __launch_bounds__(256)
collect_candidates_nib_warp_kernel(const uint4 *__restrict__ nib, int64_t n, int dim, int wd, const uint32_t *__restrict__ q, int wq,
                                   uint32_t threshold, int64_t *__restrict__ ids_out, int64_t cap, unsigned long long *__restrict__ counts) {
    constexpr int W = 4 * C;            // uint4 per document
    constexpr int DPL = 32 / W;         // documents per 512-byte load
    static_assert(32 % W == 0, "row length must divide a warp load");
    const int lane = threadIdx.x & 31;
    const int g = lane % W;
    const int Aq = (1 << wq) - 1, Ad = (1 << wd) - 1;
    // this lane's weights (group g) and the query constant Dq = Ad * sum(y)
    uint32_t w[8];
    int sy_mine = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        const int e = x >> 1, hi = x & 1;
        uint32_t packed = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int d = 32 * g + 8 * j + 4 * hi + e;
            if (d < dim) {
                int y = 0;
                for (int jq = 0; jq < wq; ++jq) y |= static_cast<int>((__ldg(q + jq * W + (d >> 5)) >> (d & 31)) & 1u) << jq;
                sy_mine += y;
                packed |= (static_cast<uint32_t>(2 * y - Aq) & 0xFFu) << (8 * j);
            }
        }
        w[x] = packed;
    }
    int sy = sy_mine;  // sum over the W groups = over the lanes of one document
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) sy += __shfl_xor_sync(0xffffffffu, sy, o);
    const int dq = Ad * sy;
    const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t n_b = (n + 31) >> 5;  // bundles of 32 documents (the nibble layout is padded to whole bundles)
    for (int64_t b = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < n_b; b += warps) {
        const uint4 *base = nib + b * 32 * W;
        uint4 v[W];
#pragma unroll
        for (int i = 0; i < W; ++i) v[i] = __ldg(base + i * 32 + lane);
#pragma unroll
        for (int i = 0; i < W; ++i) {
            int acc = 0;
            acc = umma::dp4a_su(w[0], v[i].x & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w[1], (v[i].x >> 4) & 0x0F0F0F0Fu, acc);
            acc = umma::dp4a_su(w[2], v[i].y & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w[3], (v[i].y >> 4) & 0x0F0F0F0Fu, acc);
            acc = umma::dp4a_su(w[4], v[i].z & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w[5], (v[i].z >> 4) & 0x0F0F0F0Fu, acc);
            acc = umma::dp4a_su(w[6], v[i].w & 0x0F0F0F0Fu, acc); acc = umma::dp4a_su(w[7], (v[i].w >> 4) & 0x0F0F0F0Fu, acc);
#pragma unroll
            for (int o = W / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const int64_t doc = b * 32 + i * DPL + lane / W;
            const bool hit = g == 0 && doc < n && static_cast<uint32_t>(dq - acc) <= threshold;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) {
                unsigned long long pos0 = 0;
                if (lane == 0) pos0 = atomicAdd(counts, static_cast<unsigned long long>(__popc(m)));
                pos0 = __shfl_sync(0xffffffffu, pos0, 0);
                const int64_t pos = static_cast<int64_t>(pos0) + __popc(m & ((1u << lane) - 1u));
                if (hit && ids_out && pos < cap) ids_out[pos] = doc;
            }
        }
    }
}

}  // namespace sel
