// xfbq_mma.cuh -- integer-MMA scan engine (included by xfbq_b200.cu).
//
// The XOR/popcount distance (_kernels.py:56-69) is algebraically an integer dot product of the
// codes: per dimension  sum_{i,j} 2^(i+j) (x_i ^ y_j) = Aq*x + Ad*y - 2*x*y  with
// Aq = 2^wq-1, Ad = 2^wd-1, so
//     d(doc, query) = Ad * sum_k y_k  -  sum_k x_k * (2*y_k - Aq)  =  Dq - acc
// (exact in int32; padding dimensions have x_k = 0 and contribute nothing).  `acc` is a
// u8 x s8 dot product, which the int8 tensor path (mma.sync.m16n8k32 -> IMMA.16832) computes
// ~60x faster than the POPC pipe can popcount the 16 plane pairs (profiles/microbench_r1.jsonl:
// XU/POPC 4.5 T lane-ops/s vs IMMA 568 T MAC/s).  Results are bit-identical to the POPC form.
//
// Data flow per warp (no block-level synchronisation anywhere):
//   * queries: 16*MT query rows live in registers as A fragments (s8 weights 2y-Aq, laid out by
//     mma_prep_queries_kernel in exactly the K-order the document side produces);
//   * documents: 8-doc tiles are read straight from the bit-plane bundle layout (one 128-byte
//     line per plane chunk per tile), transposed in registers from bit planes to one byte per
//     dimension (4x4 bit-block transpose by delta swaps + nibble split) and used as B fragments;
//   * selection: the accumulator is initialised to -tau_q, so "distance <= threshold" is the
//     sign bit of the result; one AND-reduction + vote per 8*NT x 16*MT scores decides whether
//     the (rare) slow path runs, which appends (distance<<32 | row id) keys to a warp-private
//     candidate list, compacted by a warp-level bitonic sort when full (search.py:129-131 order).
#pragma once

namespace mma {

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;
constexpr int TAU_OPEN = -(1 << 30);  // threshold that lets every score through (no list yet)

struct Params {
    const uint32_t *db;     // bundle layout viewed as 32-bit words
    int64_t n;              // real documents
    int64_t row_offset;
    const uint32_t *qop;    // [nq_pad][4C k-steps][4 t][2] words of 4 s8 weights
    const int32_t *qconst;  // [nq_pad] Dq = Ad * sum(y)
    uint64_t *lists;        // [ctas * WARPS][16*MT][cap] candidate lists
    uint64_t *out;          // [parts][nq][k]
    int64_t nq;
    int64_t total_iters;    // ceil(n_pad / (8*NT))
    int64_t iters_per_split;
    int k, cap, QW, DW;
};

// ------------------------------------------------------------------------------ query operand
// One warp per (padded) query row: bit-plane query words -> s8 weights 2*y - Aq in MMA K-order,
// and Dq = Ad * sum_k y_k.  Operand word ow = (s*4 + t)*2 + hi holds bytes j=0..3 for dimension
//   dim = 32C*t + 32*(s>>2) + 8*j + (s&3) + 4*hi.
__global__ void __launch_bounds__(256)
prep_queries_kernel(const uint32_t *__restrict__ q, int64_t nq, int64_t nq_pad, int dim, int wq, int wd,
                    int C, uint32_t *__restrict__ qop, int32_t *__restrict__ qconst) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= nq_pad) return;
    const int W = 4 * C;
    const int Aq = (1 << wq) - 1, Ad = (1 << wd) - 1;
    int sy = 0;
    for (int ow = lane; ow < 32 * C; ow += 32) {
        const int hi = ow & 1, t = (ow >> 1) & 3, s = ow >> 3;
        const int h = s >> 2, e = s & 3;
        uint32_t packed = 0;
        if (row < nq) {
            const int word = C * t + h;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int bit = 8 * j + e + 4 * hi;
                const int d = 32 * word + bit;
                int y = 0;
                for (int jq = 0; jq < wq; ++jq) y |= static_cast<int>((q[(row * wq + jq) * W + word] >> bit) & 1u) << jq;
                int w = 0;
                if (d < dim) { w = 2 * y - Aq; sy += y; }
                packed |= (static_cast<uint32_t>(w) & 0xFFu) << (8 * j);
            }
        }
        qop[row * (32 * C) + ow] = packed;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sy += __shfl_xor_sync(0xffffffffu, sy, o);
    if (lane == 0) qconst[row] = (row < nq) ? Ad * sy : 0;
}

// ------------------------------------------------------------------------------ bit planes -> bytes
// 4 plane words (32 dims) -> 8 words of 4 bytes: out[2e + hi] byte j = code of dim 8j + e + 4hi.
template <int WD>
__device__ __forceinline__ void planes_to_bytes(const uint32_t (&pin)[4], uint32_t (&out)[8]) {
    uint32_t p0 = pin[0], p1 = WD > 1 ? pin[1] : 0u, p2 = WD > 2 ? pin[2] : 0u, p3 = WD > 3 ? pin[3] : 0u;
    uint32_t t;
    // 2x2 bit-block transposes inside each 4x4 block (rows = planes, columns = dims mod 4)
    t = ((p0 >> 1) ^ p1) & 0x55555555u; p1 ^= t; p0 ^= t << 1;
    if (WD > 2) { t = ((p2 >> 1) ^ p3) & 0x55555555u; p3 ^= t; p2 ^= t << 1; }
    t = ((p0 >> 2) ^ p2) & 0x33333333u; p2 ^= t; p0 ^= t << 2;
    t = ((p1 >> 2) ^ p3) & 0x33333333u; p3 ^= t; p1 ^= t << 2;
    // now word p_e, nibble m = code of dim 4m + e; split even/odd nibbles into bytes
    out[0] = p0 & 0x0F0F0F0Fu; out[1] = (p0 >> 4) & 0x0F0F0F0Fu;
    out[2] = p1 & 0x0F0F0F0Fu; out[3] = (p1 >> 4) & 0x0F0F0F0Fu;
    out[4] = p2 & 0x0F0F0F0Fu; out[5] = (p2 >> 4) & 0x0F0F0F0Fu;
    out[6] = p3 & 0x0F0F0F0Fu; out[7] = (p3 >> 4) & 0x0F0F0F0Fu;
}

// D = A(s8, 16x32 row) * B(u8, 32x8 col) + C
__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                     int c0, int c1, int c2, int c3) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};\n"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}

// Quarter-row load: the C plane words (32C dims) lane t of a tile owns.
template <int C>
__device__ __forceinline__ void load_quarter(const uint32_t *base, uint32_t (&w)[C]);
template <>
__device__ __forceinline__ void load_quarter<1>(const uint32_t *base, uint32_t (&w)[1]) {
    w[0] = __ldg(base);
}
template <>
__device__ __forceinline__ void load_quarter<2>(const uint32_t *base, uint32_t (&w)[2]) {
    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(base));
    w[0] = v.x; w[1] = v.y;
}
template <>
__device__ __forceinline__ void load_quarter<4>(const uint32_t *base, uint32_t (&w)[4]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(base));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    const uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Warp-level bitonic sort of P (power of two) keys in this warp's shared scratch.
__device__ __forceinline__ void warp_bitonic(uint64_t *s, int P, int lane) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < (P >> 1); t += 32) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = s[lo], b = s[hi];
                if ((a > b) == up) { s[lo] = b; s[hi] = a; }
            }
            __syncwarp();
        }
}

// Per-lane selection state: lane l owns query row l of the warp.
struct LaneState {
    uint64_t thr_key;  // k-th best key so far (KEY_INF until k candidates exist)
    int dq;            // Dq
    int tau;           // pass iff acc >= tau  (tau = Dq - distance(thr_key))
    int count;         // entries in this row's list
};

// Sort list row `ql` (cnt entries) through the scratch, keep the k best, refresh the threshold.
// Warp-uniform arguments.  Returns the new count; writes the new -tau to *negtau_out.
__device__ __forceinline__ int compact_row(uint64_t *list_row, uint64_t *scratch, int cnt, int k, int ql,
                                           int lane, LaneState &st, int *negtau_out) {
    __syncwarp();
    int P = 2;
    while (P < cnt) P <<= 1;
    for (int i = lane; i < P; i += 32) scratch[i] = i < cnt ? __ldcg(list_row + i) : KEY_INF;
    __syncwarp();
    warp_bitonic(scratch, P, lane);
    const int keep = cnt < k ? cnt : k;
    for (int i = lane; i < keep; i += 32) list_row[i] = scratch[i];
    const uint64_t new_thr = cnt >= k ? scratch[k - 1] : KEY_INF;
    __syncwarp();
    if (lane == ql) {
        st.thr_key = new_thr;
        st.count = keep;
        if (cnt >= k) st.tau = st.dq - static_cast<int>(new_thr >> 32);
    }
    *negtau_out = -__shfl_sync(0xffffffffu, st.tau, ql);
    return keep;
}

template <int WD, int C, int MT, int NT>
__global__ void __launch_bounds__(THREADS, 1) scan_kernel(const Params p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int QPW = 16 * MT;   // query rows per warp
    constexpr int KS = 4 * C;      // k-steps of 32 dims
    constexpr int TILE = 8 * NT;   // documents per iteration
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int qw = warp % p.QW, dw = warp / p.QW;
    const int64_t q0 = (static_cast<int64_t>(blockIdx.y) * p.QW + qw) * QPW;
    if (q0 >= p.nq) return;  // no block-level synchronisation in this kernel
    uint64_t *scratch = reinterpret_cast<uint64_t *>(smem_raw) + static_cast<size_t>(warp) * p.cap;
    const int64_t cta = static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x;
    uint64_t *lists = p.lists + (cta * WARPS + warp) * QPW * static_cast<int64_t>(p.cap);

    // ---- A fragments: this warp's query rows, resident for the whole scan
    uint32_t a[MT][KS][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const uint2 r0 = __ldg(reinterpret_cast<const uint2 *>(p.qop + ((q0 + 16 * mt + g) * KS + s) * 8 + t * 2));
            const uint2 r1 = __ldg(reinterpret_cast<const uint2 *>(p.qop + ((q0 + 16 * mt + g + 8) * KS + s) * 8 + t * 2));
            a[mt][s][0] = r0.x; a[mt][s][1] = r1.x; a[mt][s][2] = r0.y; a[mt][s][3] = r1.y;
        }

    // ---- selection state: lane l <-> query row l
    LaneState st;
    {
        const int64_t myq = q0 + lane;
        const bool valid = lane < QPW && myq < p.nq;
        st.dq = valid ? p.qconst[myq] : 0;
        st.tau = valid ? TAU_OPEN : 1;  // rows without a query: acc = 0 < 1 never passes
        st.thr_key = KEY_INF;
        st.count = 0;
    }
    int negtau[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        negtau[mt][0] = -__shfl_sync(0xffffffffu, st.tau, 16 * mt + g);
        negtau[mt][1] = -__shfl_sync(0xffffffffu, st.tau, 16 * mt + g + 8);
    }

    const int64_t it_begin = static_cast<int64_t>(blockIdx.x) * p.iters_per_split;
    const int64_t it_end = min(p.total_iters, it_begin + p.iters_per_split);

    // lane (g, t) of tile nt reads, for every plane, the C words [C*t, C*t+C) of document 8*nt+g
    auto tile_ptr = [&](int64_t it, int nt, int i) -> const uint32_t * {
        const int64_t doc = it * TILE + 8 * nt + g;
        const int64_t b = doc >> 5;
        const int dl = static_cast<int>(doc & 31);
        const int word = C * t;  // first word of the quarter within the plane's 4C words
        return p.db + ((((b * WD + i) * C + (word >> 2)) * 32 + dl) << 2) + (word & 3);
    };

    uint32_t pw[NT][WD][C];
    int64_t it = it_begin + dw;
    if (it < it_end) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < WD; ++i) load_quarter<C>(tile_ptr(it, nt, i), pw[nt][i]);
    }

    for (; it < it_end; it += p.DW) {
        // ---- bit planes -> byte operands for this iteration
        uint32_t bw[NT][C][8];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < C; ++h) {
                uint32_t pin[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) pin[i] = i < WD ? pw[nt][i < WD ? i : 0][h] : 0u;
                planes_to_bytes<WD>(pin, bw[nt][h]);
            }
        // ---- prefetch the next iteration's plane words
        const int64_t itn = it + p.DW;
        if (itn < it_end) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < WD; ++i) load_quarter<C>(tile_ptr(itn, nt, i), pw[nt][i]);
        }
        // ---- acc' = sum_k x_k (2 y_k - Aq) - tau   (k-step s uses quarter words 2s, 2s+1)
        int c[MT][NT][4];
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const uint32_t b0 = bw[nt][s >> 2][2 * (s & 3)], b1 = bw[nt][s >> 2][2 * (s & 3) + 1];
                    if (s == 0) imma(c[mt][nt], a[mt][s], b0, b1, negtau[mt][0], negtau[mt][0], negtau[mt][1], negtau[mt][1]);
                    else imma(c[mt][nt], a[mt][s], b0, b1, c[mt][nt][0], c[mt][nt][1], c[mt][nt][2], c[mt][nt][3]);
                }
        // ---- any score with acc' >= 0 ?  (sign bit of the AND of all results is clear)
        int all = -1;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) all &= c[mt][nt][0] & c[mt][nt][1] & c[mt][nt][2] & c[mt][nt][3];
        if (__any_sync(0xffffffffu, all >= 0)) {
            // slow path: hits are handled one at a time with warp-uniform control flow.  The scores
            // of this iteration were biased with the thresholds in force when it started, so a
            // compaction in here must not change how they are decoded.
            const int tau_iter = st.tau;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        unsigned m = __ballot_sync(0xffffffffu, c[mt][nt][j] >= 0);
                        while (m) {
                            const int L = __ffs(m) - 1;
                            m &= m - 1;
                            const int accp = __shfl_sync(0xffffffffu, c[mt][nt][j], L);
                            const int ql = 16 * mt + (L >> 2) + 8 * (j >> 1);
                            const int64_t doc = it * TILE + 8 * nt + 2 * (L & 3) + (j & 1);
                            const int tau_q = __shfl_sync(0xffffffffu, tau_iter, ql);
                            const int dq_q = __shfl_sync(0xffffffffu, st.dq, ql);
                            const uint64_t thr = shfl_u64(st.thr_key, ql);
                            const uint32_t dist = static_cast<uint32_t>(dq_q - (accp + tau_q));
                            const uint64_t key = (static_cast<uint64_t>(dist) << 32) | static_cast<uint64_t>(p.row_offset + doc);
                            if (doc < p.n && key < thr) {
                                int cnt = __shfl_sync(0xffffffffu, st.count, ql);
                                uint64_t *row = lists + static_cast<int64_t>(ql) * p.cap;
                                if (lane == 0) row[cnt] = key;
                                ++cnt;
                                if (cnt == p.cap) {
                                    int nv;
                                    cnt = compact_row(row, scratch, cnt, p.k, ql, lane, st, &nv);
#pragma unroll
                                    for (int m2 = 0; m2 < MT; ++m2) {
                                        if (16 * m2 + g == ql) negtau[m2][0] = nv;
                                        if (16 * m2 + g + 8 == ql) negtau[m2][1] = nv;
                                    }
                                } else if (lane == ql) {
                                    st.count = cnt;
                                }
                            }
                        }
                    }
        }
    }

    // ---- emit: every query row of this warp, sorted, KEY_INF padded
    const int64_t part = static_cast<int64_t>(blockIdx.x) * p.DW + dw;
    for (int ql = 0; ql < QPW; ++ql) {
        const int64_t q = q0 + ql;
        if (q >= p.nq) break;
        const int cnt = __shfl_sync(0xffffffffu, st.count, ql);
        uint64_t *row = lists + static_cast<int64_t>(ql) * p.cap;
        __syncwarp();
        int P = 2;
        while (P < cnt) P <<= 1;
        for (int i = lane; i < P; i += 32) scratch[i] = i < cnt ? __ldcg(row + i) : KEY_INF;
        __syncwarp();
        warp_bitonic(scratch, P, lane);
        uint64_t *dst = p.out + (part * p.nq + q) * p.k;
        for (int i = lane; i < p.k; i += 32) dst[i] = (i < cnt && i < P) ? scratch[i] : KEY_INF;
        __syncwarp();
    }
}

}  // namespace mma
