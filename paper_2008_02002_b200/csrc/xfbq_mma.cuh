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
// Data flow of one CTA (8 warps; lane 0 of warp 0 also issues the TMA copies), per stage of 8 iterations x TILE =
// 8*NT documents (whole bundles, contiguous in HBM, fetched by one cp.async.bulk per stage):
//   * queries: 16*MT query rows per warp live in registers as A fragments (s8 weights 2y-Aq,
//     laid out by prep_queries_kernel in exactly the K-order the document side produces);
//   * documents: the engine streams the nibble layout (row-major 4-bit codes derived from the
//     bit planes by planes_to_nibbles_kernel); warp w reads iteration w of the raw stage from
//     shared memory, splits nibbles into bytes (3 ALU ops per 8 dims) and stores the B fragments
//     to a ring of byte stages, so a tile is unpacked once per CTA however many warps consume it;
//   * every (query-warp, doc-warp) consumes its iterations of the stage: 8 LDS.128 + MT*NT*4C
//     IMMAs; the accumulator is initialised to -tau_q, so "distance <= threshold" is the sign
//     bit of the result and one AND-reduction + vote per TILE x 16*MT scores decides whether the
//     (rare) slow path runs; there, lanes append (distance<<32 | row id) keys to the warp's
//     candidate lists in parallel (shared-memory counters), and rows that could overflow in the
//     next iteration are compacted by a warp-level bitonic sort (search.py:129-131 order);
//   * work = groups x stages is linearised and cut into gridDim.x equal ranges, so every CTA
//     scans the same number of stages and a query group is split over as few CTAs as possible.
#pragma once

namespace mma {

constexpr int WARPS = 8;        // warps per CTA in ring (batch) mode and the default fused mode
constexpr int WARPS_WIDE = 16;  // fused mode for <= 16 queries: twice the warps hide ALU latency
constexpr int WARPS_BATCH = 12; // ring mode with >= 12 query warps: 3 warps per scheduler
constexpr int TAU_OPEN = -(1 << 30);  // threshold that lets every score through (no list yet)


struct Params {
    const void *db;           // nibble layout: row-major, 64C bytes per document (see planes_to_nibbles_kernel)
    int64_t n;                // real documents
    int64_t n_pad;            // documents the buffer holds (multiple of 32)
    int64_t row_offset;
    const uint32_t *qop;      // [nq_pad/16][4C k-steps][32 lanes][4] A fragments (s8 weights)
    const int32_t *qconst;    // [nq_pad] Dq = Ad * sum(y)
    const int32_t *tau_init;  // [nq] initial thresholds (acc domain) or nullptr
    uint64_t *lists;          // [gridDim.x * WARPS][16*MT][cap] candidate lists
    uint64_t *out;            // [slots * DW][nq][k], pre-filled with KEY_INF
    int64_t nq;
    int64_t stages;           // ceil(n_pad / (STAGE_ITERS * TILE))
    int groups;               // query groups of QW * 16*MT queries
    int k, cap, QW, DW;
    int RR, BR;               // ring depths: raw (TMA) stages, byte (B fragment) stages
};

// ------------------------------------------------------------------------------ query operand
// One warp per (padded) query row: bit-plane query words -> s8 weights 2*y - Aq in MMA K-order,
// and Dq = Ad * sum_k y_k.  Operand word ow = (s*4 + t)*2 + hi holds bytes j=0..3 for dimension
//   dim = 32C*t + 32*(s>>2) + 8*j + (s&3) + 4*hi; words are stored in mma A-fragment order so a
// lane fetches the four registers of one (16-row tile, k-step) with a single 128-bit load.
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
        // fragment order: 16-row tile, k-step, lane (g = row%8, t), register (a0..a3 = half + 2*hi)
        const int64_t tile = row >> 4;
        const int rr = static_cast<int>(row & 15);
        qop[((tile * (4 * C) + s) * 32 + (rr & 7) * 4 + t) * 4 + (rr >> 3) + 2 * hi] = packed;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sy += __shfl_xor_sync(0xffffffffu, sy, o);
    if (lane == 0) qconst[row] = (row < nq) ? Ad * sy : 0;
}

// ------------------------------------------------------------------------------ bit planes -> nibbles
// The tensor engine streams a derived copy of the database: row-major 4-bit codes ("nibble
// layout"), 64C bytes per document, one uint4 per group of 32 dims; word e of a group holds, in
// nibble m, the code of dim 4m + e.  That is the 4x4 bit-block transpose of the group's (up to) 4
// plane words, done with delta swaps; unpacking to MMA bytes is then 3 ALU ops per 8 dims.
__device__ __forceinline__ uint4 planes_to_nibbles(uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3) {
    uint32_t t;
    t = ((p0 >> 1) ^ p1) & 0x55555555u; p1 ^= t; p0 ^= t << 1;
    t = ((p2 >> 1) ^ p3) & 0x55555555u; p3 ^= t; p2 ^= t << 1;
    t = ((p0 >> 2) ^ p2) & 0x33333333u; p2 ^= t; p0 ^= t << 2;
    t = ((p1 >> 2) ^ p3) & 0x33333333u; p3 ^= t; p1 ^= t << 2;
    return make_uint4(p0, p1, p2, p3);
}

// bundle layout (bit planes) -> nibble layout; one thread per (document, 32-dim group).
__global__ void __launch_bounds__(256)
planes_to_nibbles_kernel(const uint32_t *__restrict__ db, int64_t n_pad, int wd, int C, uint4 *__restrict__ out) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int G = 4 * C;  // 32-dim groups per document
    if (e >= n_pad * G) return;
    // consecutive threads take consecutive documents of one group: coalesced reads of the bundle layout
    const int64_t tile = e / (32 * G);
    const int rem = static_cast<int>(e - tile * (32 * G));
    const int grp = rem >> 5, dl = rem & 31;
    const int64_t b = tile;  // bundle
    uint32_t p[4] = {0u, 0u, 0u, 0u};
    for (int i = 0; i < wd; ++i) p[i] = db[((((b * wd + i) * C + (grp >> 2)) * 32 + dl) << 2) + (grp & 3)];
    out[(b * 32 + dl) * G + grp] = planes_to_nibbles(p[0], p[1], p[2], p[3]);
}

// nibble layout -> bundle layout (bit planes): the 4x4 bit-block transpose is its own inverse.  Lets a server that only answers
// single queries keep the nibbles alone (1x the packed size) and rebuild the packed codes when something needs them.
__global__ void __launch_bounds__(256)
nibbles_to_planes_kernel(const uint4 *__restrict__ nib, int64_t n_pad, int wd, int C, uint32_t *__restrict__ db) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int G = 4 * C;
    if (e >= n_pad * G) return;
    const int64_t b = e / (32 * G);
    const int rem = static_cast<int>(e - b * (32 * G));
    const int grp = rem >> 5, dl = rem & 31;
    const uint4 w = nib[(b * 32 + dl) * G + grp];
    const uint4 p = planes_to_nibbles(w.x, w.y, w.z, w.w);
    const uint32_t pl[4] = {p.x, p.y, p.z, p.w};
    for (int i = 0; i < wd; ++i) db[((((b * wd + i) * C + (grp >> 2)) * 32 + dl) << 2) + (grp & 3)] = pl[i];
}

// D = A(s8, 16x32 row) * B(u8, 32x8 col) + C
__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                     int c0, int c1, int c2, int c3) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};\n"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    const uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Per-lane selection state: lane l owns query row l of the warp.
struct LaneState {
    int dq;   // Dq = Ad * sum(y) of the row's query
    int tau;  // pass iff acc >= tau  (tau = Dq - distance of the k-th best key so far)
};

// Warp-level radix select, in place on a candidate list row in global memory (read through L2):
// keeps exactly the k smallest of the cnt > k unique keys (order not preserved) and returns the
// k-th smallest key.  MSB-first, one byte per pass, starting at the highest byte in which the keys
// differ; 256-bin histogram per warp in shared memory.  Cost ~ (passes + 2) * cnt / 32 loads per
// lane, instead of a cnt * log^2(cnt) sort.
__device__ __noinline__ uint64_t select_row(uint64_t *row, int cnt, int k, int *hist, int lane) {
    __syncwarp();
    const uint64_t first = __ldcg(row);
    uint64_t diff = 0;
    for (int i = lane; i < cnt; i += 32) diff |= __ldcg(row + i) ^ first;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(diff), o);
        const uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(diff >> 32), o);
        diff |= (static_cast<uint64_t>(hi) << 32) | lo;
    }
    int shift = ((63 - __clzll(static_cast<long long>(diff | 1ull))) >> 3) << 3;  // byte holding the top differing bit
    uint64_t hi_mask = shift + 8 >= 64 ? 0ull : ~((1ull << (shift + 8)) - 1ull);    // bits already common to all keys
    uint64_t prefix = first & hi_mask;
    int want = k;  // rank of the k-th key inside the current candidate bucket (1-based)
    while (true) {
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) {
            const uint64_t key = __ldcg(row + i);
            if ((key & hi_mask) == prefix) atomicAdd(&hist[static_cast<int>(key >> shift) & 255], 1);
        }
        __syncwarp();
        int h[8], s = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) { h[e] = hist[8 * lane + e]; s += h[e]; }
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const int exc = inc - s;
        const bool mine = exc < want && want <= inc;  // exactly one lane
        int bucket = 0, below = exc, bcnt = 0;
        if (mine) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (bcnt == 0) {
                    if (below + h[e] >= want) { bucket = 8 * lane + e; bcnt = h[e]; }
                    else below += h[e];
                }
            }
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        bucket = __shfl_sync(0xffffffffu, bucket, src);
        below = __shfl_sync(0xffffffffu, below, src);
        bcnt = __shfl_sync(0xffffffffu, bcnt, src);
        prefix |= static_cast<uint64_t>(bucket) << shift;
        hi_mask |= 0xFFull << shift;
        want -= below;
        __syncwarp();
        if (bcnt == want || shift == 0) break;  // the whole bucket belongs to the k smallest
        shift -= 8;
    }
    // partition in place: keep keys whose fixed bits are <= prefix (exactly k of them); k-th = their max
    uint64_t kth = 0;
    int out = 0;
    for (int base = 0; base < cnt; base += 32) {
        const int i = base + lane;
        const uint64_t key = i < cnt ? __ldcg(row + i) : KEY_INF;
        const bool keep = i < cnt && (key & hi_mask) <= prefix;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            row[out + __popc(m & ((1u << lane) - 1u))] = key;  // out + rank <= i: never overwrites unread keys
            kth = key > kth ? key : kth;
        }
        out += __popc(m);
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(kth), o);
        const uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(kth >> 32), o);
        const uint64_t other = (static_cast<uint64_t>(hi) << 32) | lo;
        kth = other > kth ? other : kth;
    }
    __syncwarp();
    return kth;
}

// Warp-level bitonic sort of P (power of two) keys in this warp's shared scratch (small lists).
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

// Small lists (cap <= 512): sort the row through the warp's shared scratch, keep the k best.
__device__ __noinline__ int compact_row_sorted(uint64_t *list_row, uint64_t *scratch, int *cnt_p, int k, int ql,
                                               int lane, int dq, int *tau_io) {
    __syncwarp();
    const int cnt = *cnt_p;
    int P = 2;
    while (P < cnt) P <<= 1;
    for (int i = lane; i < P; i += 32) scratch[i] = i < cnt ? __ldcg(list_row + i) : KEY_INF;
    __syncwarp();
    warp_bitonic(scratch, P, lane);
    const int keep = cnt < k ? cnt : k;
    for (int i = lane; i < keep; i += 32) list_row[i] = scratch[i];
    const uint64_t kth = cnt >= k ? scratch[k - 1] : KEY_INF;
    __syncwarp();
    int tau = *tau_io;
    if (lane == ql) {
        *cnt_p = keep;
        if (cnt >= k) tau = dq - static_cast<int>(kth >> 32);
    }
    *tau_io = tau;
    __syncwarp();
    return -__shfl_sync(0xffffffffu, tau, ql);
}

// Cut list row `ql` to its k best keys and refresh the row's threshold.  Warp-uniform call.
// Returns -tau of the row (for the per-lane accumulator bias copies).
__device__ __noinline__ int compact_row(uint64_t *list_row, int *hist, int *cnt_p, int k, int ql, int lane,
                                        int dq, int *tau_io) {
    __syncwarp();
    const int cnt = *cnt_p;
    int tau = *tau_io;
    if (cnt > k) {
        const uint64_t kth = select_row(list_row, cnt, k, hist, lane);
        if (lane == ql) {
            *cnt_p = k;
            tau = dq - static_cast<int>(kth >> 32);
        }
    }
    *tau_io = tau;
    __syncwarp();
    return -__shfl_sync(0xffffffffu, tau, ql);
}

// Out-of-line candidate push for one 16-row x 8-doc tile (keeps the cold code out of the hot loop's
// instruction-cache footprint): lanes whose score passed append (distance << 32 | row id).
__device__ __noinline__ void push_tile(int v0, int v1, int v2, int v3, int dq0, int dq1, int nt0, int nt1,
                                       uint32_t doc_a, uint32_t n_docs, int row_a, uint64_t row_offset,
                                       uint64_t *lists, int *cnt_s, int cap) {
    // (v0, v1): row row_a, docs doc_a, doc_a+1;  (v2, v3): row row_a+8, same docs
    const int v[4] = {v0, v1, v2, v3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t doc = doc_a + (j & 1);
        if (v[j] >= 0 && doc < n_docs) {
            const int row = row_a + 8 * (j >> 1);
            const uint32_t dist = static_cast<uint32_t>((j >> 1 ? dq1 + nt1 : dq0 + nt0) - v[j]);
            const int pos = atomicAdd(&cnt_s[row], 1);
            lists[row * cap + pos] = (static_cast<uint64_t>(dist) << 32) | (row_offset + doc);
        }
    }
}

// ------------------------------------------------------------------------------ mbarrier / TMA
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// The retry loop lives inside the asm block: around a C++ loop the compiler puts a YIELD in front of every try_wait,
// the first one included, and a warp whose barrier has already completed still hands its issue slot away.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
// TMA bulk copy global -> shared (1-D, contiguous), completion signalled on `bar` as tx bytes.
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int AHEAD = 2;  // stages a worker transposes ahead of the stage it consumes
constexpr int SORT_CAP_MAX = 512;  // lists up to this capacity are compacted by a shared-memory sort

// Shared-memory carve-up shared by host (size) and device (pointers).
struct SmemLayout {
    uint32_t raw_off, byte_off, scratch_off, cnt_off, bar_off, total;
};
__host__ __device__ inline SmemLayout smem_layout(int raw_stage_bytes, int byte_stage_bytes, int RR, int BR, int cap, int warps) {
    SmemLayout L;
    uint32_t off = 0;
    L.raw_off = off; off += static_cast<uint32_t>(RR) * raw_stage_bytes;
    off = (off + 127u) & ~127u;
    L.byte_off = off; off += static_cast<uint32_t>(BR) * byte_stage_bytes;
    // per warp: sort scratch for small lists (cap <= 512 keys), else the radix-select histogram
    L.scratch_off = off; off += static_cast<uint32_t>(warps) * (cap <= SORT_CAP_MAX ? cap * 8 : 256 * 4);
    L.cnt_off = off; off += warps * 32 * 4;
    L.bar_off = off; off += static_cast<uint32_t>(2 * RR + 2 * BR) * 8;
    L.total = off;
    return L;
}

// Ring cursor: slot index and the mbarrier phase parity to wait on; no divisions in the hot loop.
struct Ring {
    int idx;
    uint32_t phase;
    __device__ __forceinline__ void advance(int n) {
        if (++idx == n) { idx = 0; phase ^= 1u; }
    }
};

// One CTA = 8 worker warps.
//   TMA    : this CTA's document stages stream HBM -> raw ring as bulk copies (RR deep), issued
//            by thread 0 whenever a slot has been released by all warps
//   ring mode (FUSED = false; several query warps share each document tile):
//     worker w: [transpose] its iteration slot of stage i+AHEAD: raw ring -> byte ring (B fragments)
//               [consume]   its iterations of stage i: byte ring -> IMMA -> threshold filter -> lists
//   fused mode (FUSED = true; QW == 1, every tile is consumed by exactly one warp):
//     worker w: raw ring -> registers (transpose) -> IMMA -> filter, no byte ring
// Hand-offs are mbarriers (raw_full/raw_empty, byte_full/byte_empty), so a warp that runs a list
// compaction only stalls the others once the rings' slack is used up (no per-stage block barrier).
template <int C, int MT, int NT, bool FUSED, int NW>
__global__ void __launch_bounds__(NW * 32, 1) scan_kernel(const Params p) {
    constexpr int WARPS = NW;           // shadows the namespace default
    constexpr int WARPS_DEFAULT = 8;
    constexpr int STAGE_ITERS = NW;     // iterations per stage: one produced by each warp
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int QPW = 16 * MT;        // query rows per warp
    constexpr int KS = 4 * C;           // k-steps of 32 dims
    constexpr int TILE = 8 * NT;        // documents per iteration
    constexpr int WPL = NT * C * 8;     // B-fragment words per lane per iteration
    constexpr int RCH = WPL / 4;        // 16-byte chunks per lane per iteration
    constexpr int STAGE_DOCS = STAGE_ITERS * TILE;
    constexpr int ROW_BYTES = 64 * C;                        // one document: 128C nibbles
    constexpr int RAW_STAGE_BYTES = STAGE_DOCS * ROW_BYTES;  // contiguous in HBM (nibble layout is row-major)
    constexpr int BYTE_STAGE_BYTES = STAGE_ITERS * WPL * 32 * 4;
    static_assert(STAGE_DOCS % 32 == 0, "a stage must be whole bundles");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int RR = p.RR, BR = p.BR;
    const SmemLayout L = smem_layout(RAW_STAGE_BYTES, BYTE_STAGE_BYTES, RR, BR, p.cap, NW);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + L.bar_off);
    uint64_t *raw_full = bars, *raw_empty = bars + RR, *byte_full = bars + 2 * RR, *byte_empty = bars + 2 * RR + BR;

    // ---- this CTA's share of the linearised (group, stage) work
    const int64_t T = p.stages;
    const int64_t W = static_cast<int64_t>(p.groups) * T;
    const int64_t G = gridDim.x;
    const int64_t lin_begin = static_cast<int64_t>(blockIdx.x) * W / G;
    const int64_t lin_end = (static_cast<int64_t>(blockIdx.x) + 1) * W / G;
    const int S = static_cast<int>(lin_end - lin_begin);  // stages this CTA streams
    const int gr_begin = static_cast<int>(lin_begin / T);
    const int sd_begin = static_cast<int>(lin_begin - static_cast<int64_t>(gr_begin) * T);
    const int Ti = static_cast<int>(T);

    if (threadIdx.x == 0) {
        for (int i = 0; i < RR; ++i) { mbar_init(&raw_full[i], 1); mbar_init(&raw_empty[i], WARPS); }
        for (int i = 0; i < BR; ++i) { mbar_init(&byte_full[i], WARPS); mbar_init(&byte_empty[i], WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // ---- TMA issue, folded into warp 0 / lane 0: whenever it passes by (and while it spins on a
    // barrier) it refills every raw-ring slot that all warps have released.  A 9th issuer warp
    // would cap the kernel at 168 registers per thread (register file is carved per 4 warps).
    const int64_t db_bytes = p.n_pad * static_cast<int64_t>(ROW_BYTES);
    Ring is_ring{0, 1u};  // "empty" waits start on the phase that counts as already completed
    int is_sd = sd_begin, issued = 0;
    auto pump = [&]() {
        if (threadIdx.x != 0) return;
        while (issued < S && mbar_test(&raw_empty[is_ring.idx], is_ring.phase)) {
            const int64_t off = static_cast<int64_t>(is_sd) * RAW_STAGE_BYTES;
            int64_t bytes = db_bytes - off;
            if (bytes > RAW_STAGE_BYTES) bytes = RAW_STAGE_BYTES;
            mbar_arrive_expect_tx(&raw_full[is_ring.idx], static_cast<uint32_t>(bytes));
            tma_bulk_g2s(smem_raw + L.raw_off + static_cast<size_t>(is_ring.idx) * RAW_STAGE_BYTES,
                         reinterpret_cast<const unsigned char *>(p.db) + off, static_cast<uint32_t>(bytes), &raw_full[is_ring.idx]);
            is_ring.advance(RR);
            if (++is_sd == Ti) is_sd = 0;
            ++issued;
        }
    };
    auto wait_bar = [&](uint64_t *bar, uint32_t parity) {  // warp 0 keeps the TMA ring fed while it waits
        if (warp == 0) {
            while (!mbar_test(bar, parity)) pump();
        } else {
            mbar_wait(bar, parity);
        }
    };
    pump();

    // ================================ worker warps ================================
    const int g = lane >> 2, t = lane & 3;
    const int qw = FUSED ? 0 : warp % p.QW, dw = FUSED ? warp : warp / p.QW;
    const int DW = FUSED ? WARPS : p.DW;
    const bool small_lists = p.cap <= SORT_CAP_MAX;  // sorted (bitonic) vs selected (radix) compaction / emission
    uint64_t *scratch = reinterpret_cast<uint64_t *>(smem_raw + L.scratch_off) + static_cast<size_t>(warp) * p.cap;
    int *hist = reinterpret_cast<int *>(smem_raw + L.scratch_off) + warp * 256;
    int *cnt_s = reinterpret_cast<int *>(smem_raw + L.cnt_off) + warp * 32;
    uint64_t *lists = p.lists + (static_cast<int64_t>(blockIdx.x) * WARPS + warp) * QPW * static_cast<int64_t>(p.cap);

    // raw stage -> nibble words of this warp's iteration slot: lane (g, t) owns the quarter
    // [32C*t, 32C*(t+1)) of document warp*TILE + 8*nt + g, i.e. C groups of 32 dims = C uint4
    auto load_nibbles = [&](int r, uint4 (&nw)[NT][C]) {
        const uint4 *raw = reinterpret_cast<const uint4 *>(smem_raw + L.raw_off + static_cast<size_t>(r) * RAW_STAGE_BYTES);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < C; ++h) nw[nt][h] = raw[(warp * TILE + 8 * nt + g) * (4 * C) + C * t + h];
    };
    // nibble word e of a group holds, in nibble m, the code of dim 4m + e; even / odd nibbles split
    // into the two byte words of k-step 4h + e: byte j = dim 8j + e (+4)
    auto nibbles_to_fragments = [&](const uint4 (&nw)[NT][C], uint32_t (&bw)[WPL]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < C; ++h) {
                const uint32_t w[4] = {nw[nt][h].x, nw[nt][h].y, nw[nt][h].z, nw[nt][h].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    bw[(nt * C + h) * 8 + 2 * e] = w[e] & 0x0F0F0F0Fu;
                    bw[(nt * C + h) * 8 + 2 * e + 1] = (w[e] >> 4) & 0x0F0F0F0Fu;
                }
            }
    };

    // per-segment state
    int64_t q0 = 0, part = 0;
    bool has_q = false;
    uint32_t a[MT][KS][4];
    LaneState st;
    st.dq = 0; st.tau = 1;
    int negtau[MT][2], dqrow[MT][2];

    auto emit_segment = [&]() {  // every query row of this warp: its <= k best keys, KEY_INF padded
        if (!has_q) return;        // (sorted for small lists, unsorted otherwise: the merge sorts those)
        __syncwarp();
        for (int ql = 0; ql < QPW; ++ql) {
            const int64_t q = q0 + ql;
            if (q >= p.nq) break;
            int cnt = cnt_s[ql];
            uint64_t *row = lists + static_cast<int64_t>(ql) * p.cap;
            uint64_t *dst = p.out + (part * p.nq + q) * p.k;
            if (small_lists) {
                int P = 2;
                while (P < cnt) P <<= 1;
                for (int i = lane; i < P; i += 32) scratch[i] = i < cnt ? __ldcg(row + i) : KEY_INF;
                __syncwarp();
                warp_bitonic(scratch, P, lane);
                for (int i = lane; i < p.k; i += 32) dst[i] = i < cnt ? scratch[i] : KEY_INF;
                __syncwarp();
            } else {
                if (cnt > p.k) {
                    select_row(row, cnt, p.k, hist, lane);
                    cnt = p.k;
                }
                __syncwarp();
                for (int i = lane; i < p.k; i += 32) dst[i] = i < cnt ? __ldcg(row + i) : KEY_INF;
            }
        }
        __syncwarp();
    };
    auto begin_segment = [&](int gr) {
        // part slot: CTAs overlapping group gr are numbered from the first one
        int64_t c_first = (static_cast<int64_t>(gr) * T * G) / W;
        while (c_first > 0 && c_first * W / G > static_cast<int64_t>(gr) * T) --c_first;
        while ((c_first + 1) * W / G <= static_cast<int64_t>(gr) * T) ++c_first;
        part = (static_cast<int64_t>(blockIdx.x) - c_first) * DW + dw;
        q0 = (static_cast<int64_t>(gr) * (FUSED ? 1 : p.QW) + qw) * QPW;
        has_q = q0 < p.nq;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (has_q) v = __ldg(reinterpret_cast<const uint4 *>(p.qop) + (((q0 >> 4) + mt) * KS + s) * 32 + lane);
                a[mt][s][0] = v.x; a[mt][s][1] = v.y; a[mt][s][2] = v.z; a[mt][s][3] = v.w;
            }
        const int64_t myq = q0 + lane;
        const bool valid = has_q && lane < QPW && myq < p.nq;
        st.dq = valid ? p.qconst[myq] : 0;
        st.tau = valid ? (p.tau_init ? max(TAU_OPEN, p.tau_init[myq]) : TAU_OPEN) : 1;  // no query: acc = 0 < 1
        __syncwarp();
        cnt_s[lane] = 0;
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                negtau[mt][hf] = -__shfl_sync(0xffffffffu, st.tau, 16 * mt + g + 8 * hf);
                dqrow[mt][hf] = __shfl_sync(0xffffffffu, st.dq, 16 * mt + g + 8 * hf);
            }
    };

    // IMMA + threshold filter + (rare) candidate pushes for one iteration (TILE documents from doc0)
    const uint32_t n_docs = static_cast<uint32_t>(p.n);
    auto process = [&](const uint32_t (&bw)[WPL], uint32_t doc0) {
        // acc' = sum_k x_k (2 y_k - Aq) - tau; k-step s2 = 4h + e uses words (nt*C + h)*8 + 2e, +1
        int c[MT][NT][4];
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const uint32_t b0 = bw[(nt * C + (s2 >> 2)) * 8 + 2 * (s2 & 3)];
                    const uint32_t b1 = bw[(nt * C + (s2 >> 2)) * 8 + 2 * (s2 & 3) + 1];
                    if (s2 == 0) imma(c[mt][nt], a[mt][s2], b0, b1, negtau[mt][0], negtau[mt][0], negtau[mt][1], negtau[mt][1]);
                    else imma(c[mt][nt], a[mt][s2], b0, b1, c[mt][nt][0], c[mt][nt][1], c[mt][nt][2], c[mt][nt][3]);
                }
        // any score with acc' >= 0 ?  (the AND of the results has a clear sign bit); pm = per-tile ANDs
        int pm[MT][NT];
        int all = -1;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                pm[mt][nt] = (c[mt][nt][0] & c[mt][nt][1]) & (c[mt][nt][2] & c[mt][nt][3]);
                all &= pm[mt][nt];
            }
        if (__any_sync(0xffffffffu, all >= 0)) {
            // slow path: lanes append their own hits; a row gains at most TILE keys per iteration
            // and is compacted as soon as fewer than TILE slots remain
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    if (pm[mt][nt] >= 0)  // per-lane: one of this lane's 4 scores of the tile passed
                        push_tile(c[mt][nt][0], c[mt][nt][1], c[mt][nt][2], c[mt][nt][3], dqrow[mt][0], dqrow[mt][1],
                                  negtau[mt][0], negtau[mt][1], doc0 + 8 * nt + 2 * t, n_docs, 16 * mt + g,
                                  static_cast<uint64_t>(p.row_offset), lists, cnt_s, p.cap);
                }
            __syncwarp();
            unsigned need = __ballot_sync(0xffffffffu, lane < QPW && cnt_s[lane] > p.cap - TILE);
            while (need) {
                const int ql = __ffs(need) - 1;
                need &= need - 1;
                const int nv = small_lists
                                   ? compact_row_sorted(lists + ql * p.cap, scratch, &cnt_s[ql], p.k, ql, lane, st.dq, &st.tau)
                                   : compact_row(lists + ql * p.cap, hist, &cnt_s[ql], p.k, ql, lane, st.dq, &st.tau);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    if (16 * mt + g == ql) negtau[mt][0] = nv;
                    if (16 * mt + g + 8 == ql) negtau[mt][1] = nv;
                }
            }
        }
    };

    const uint32_t n_pad32 = static_cast<uint32_t>(p.n_pad);
    int gr = gr_begin, sd = sd_begin;  // consume cursor: group and document stage
    begin_segment(gr);

    if (FUSED) {
        Ring rf{0, 0u};
        for (int ci = 0; ci < S; ++ci) {
            uint4 nw[NT][C];
            uint32_t bw[WPL];
            wait_bar(&raw_full[rf.idx], rf.phase);
            load_nibbles(rf.idx, nw);
            __syncwarp();  // all lanes have their words in registers before the slot is handed back
            if (lane == 0) mbar_arrive(&raw_empty[rf.idx]);
            rf.advance(RR);
            pump();
            const uint32_t doc0 = (static_cast<uint32_t>(sd) * STAGE_ITERS + warp) * TILE;
            if (has_q && doc0 + TILE <= n_pad32) {
                nibbles_to_fragments(nw, bw);
                process(bw, doc0);
            }
            if (++sd == Ti) {
                sd = 0;
                if (ci + 1 < S) { emit_segment(); begin_segment(++gr); }
            }
        }
    } else {
        Ring tr_raw{0, 0u}, tr_byte{0, 1u}, cs{0, 0u};
        auto transpose_stage = [&]() {  // this warp's iteration slot: raw ring -> byte ring
            uint4 nw[NT][C];
            uint32_t bw[WPL];
            wait_bar(&byte_empty[tr_byte.idx], tr_byte.phase);
            wait_bar(&raw_full[tr_raw.idx], tr_raw.phase);
            load_nibbles(tr_raw.idx, nw);
            nibbles_to_fragments(nw, bw);
            uint4 *dst = reinterpret_cast<uint4 *>(smem_raw + L.byte_off + static_cast<size_t>(tr_byte.idx) * BYTE_STAGE_BYTES) +
                         static_cast<size_t>(warp) * (RCH * 32) + lane;
#pragma unroll
            for (int r = 0; r < RCH; ++r) dst[r * 32] = make_uint4(bw[4 * r], bw[4 * r + 1], bw[4 * r + 2], bw[4 * r + 3]);
            __syncwarp();  // orders every lane's reads / writes before the elected lane's release-arrive
            if (lane == 0) { mbar_arrive(&raw_empty[tr_raw.idx]); mbar_arrive(&byte_full[tr_byte.idx]); }
            tr_raw.advance(RR);
            tr_byte.advance(BR);
            pump();
        };
        for (int pi = 0; pi < AHEAD && pi < S; ++pi) transpose_stage();
        for (int ci = 0; ci < S; ++ci) {
            if (ci + AHEAD < S) transpose_stage();
            wait_bar(&byte_full[cs.idx], cs.phase);
            if (has_q) {
                // iterations dw, dw+DW, ... of the stage; fragments of the next one are fetched
                // from shared memory while the IMMAs of the current one run (two register sets)
                const uint32_t stage_doc0 = static_cast<uint32_t>(sd) * STAGE_DOCS;
                const uint32_t left = n_pad32 - stage_doc0;
                const int n_it = left >= static_cast<uint32_t>(STAGE_DOCS) ? STAGE_ITERS : static_cast<int>(left / TILE);
                const uint4 *stage_src = reinterpret_cast<const uint4 *>(smem_raw + L.byte_off + static_cast<size_t>(cs.idx) * BYTE_STAGE_BYTES) + lane;
                auto fetch = [&](uint32_t (&bw)[WPL], int i) {
                    const uint4 *src = stage_src + i * (RCH * 32);
#pragma unroll
                    for (int r = 0; r < RCH; ++r) {
                        const uint4 v = src[r * 32];
                        bw[4 * r] = v.x; bw[4 * r + 1] = v.y; bw[4 * r + 2] = v.z; bw[4 * r + 3] = v.w;
                    }
                };
                if (NW <= WARPS_DEFAULT) {
                    // two fragment register sets: the LDS of iteration i+1 overlap the IMMAs of i
                    uint32_t bwA[WPL], bwB[WPL];
                    int i = dw;
                    if (i < n_it) fetch(bwA, i);
                    while (i < n_it) {
                        const int i2 = i + DW;
                        if (i2 < n_it) fetch(bwB, i2);
                        process(bwA, stage_doc0 + i * TILE);
                        if (i2 >= n_it) break;
                        const int i3 = i2 + DW;
                        if (i3 < n_it) fetch(bwA, i3);
                        process(bwB, stage_doc0 + i2 * TILE);
                        i = i3;
                    }
                } else {
                    // more warps per scheduler instead (register budget 168): single fragment set
                    for (int i = dw; i < n_it; i += DW) {
                        uint32_t bw[WPL];
                        fetch(bw, i);
                        process(bw, stage_doc0 + i * TILE);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&byte_empty[cs.idx]);
            cs.advance(BR);
            if (++sd == Ti) {
                sd = 0;
                if (ci + 1 < S) { emit_segment(); begin_segment(++gr); }
            }
        }
    }
    emit_segment();
}

// tau_init[q] = Dq - distance(k-th key of a sample scan), or TAU_OPEN when the sample had < k rows.
__global__ void tau_from_keys_kernel(const uint64_t *__restrict__ keys, const int32_t *__restrict__ qconst,
                                     int64_t nq, int k, int32_t *__restrict__ tau) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t kth = keys[q * k + (k - 1)];
    tau[q] = kth == KEY_INF ? TAU_OPEN : qconst[q] - static_cast<int32_t>(kth >> 32);
}

}  // namespace mma
