// xfbq_umma.cuh -- tcgen05 (5th-generation tensor core) scan engine (included by xfbq_b200.cu).
//
// Same arithmetic as the IMMA engine (xfbq_mma.cuh): the XOR/popcount distance of _kernels.py:56-69
// is the exact integer form  d = Dq - sum_k x_k (2 y_k - Aq);  here the s8 x s8 -> s32 dot products
// run on tcgen05.mma.kind::i8 (measured 8 188 MAC/clk/SM, 4x the mma.sync IMMA pipe) with the
// accumulators in tensor memory.
//
// Two kernels share the loader / issuer design (one persistent CTA per SM, roles meet only at mbarriers):
//   loader (1 thread)    one cp.async.bulk per stage: the engine streams a derived "byte tile" copy of the
//                        codes -- 128 documents x 128C bytes, K-major with the 128-byte swizzle, i.e. the
//                        exact shared-memory image of a tcgen05 B operand -- so nothing touches the data
//                        between HBM/L2 and the tensor core (a CUDA-core unpack stage cost more than the MMAs)
//   issuer (1 thread)    per stage and per 128-query tile: 4C x tcgen05.mma (M = 128 queries, N = 128
//                        documents, K = 32) into one of three 128-column TMEM accumulators;
//                        tcgen05.commit releases the operand stage / publishes the accumulator
// and differ in who maintains the candidate lists:
//   scan_kernel          8 epilogue warps: tcgen05.ld of 32 lanes x 128 columns, accumulator handed back, then
//                        per 32 scores of the thread's OWN query row a 3-input max tree, one compare with the
//                        row's threshold register, one vote; hits go to thread-private lists, compacted in place
//                        (register radix select).  Used for the sample scans that seed the thresholds (every
//                        score passes at first) and for small problems.
//   scan_queue_kernel    12 stateless drain warps park passing score rows in shared-memory rings, 2 resolver
//                        warps own the lists (see the comment above that kernel).  Used for the big scans: the
//                        tensor pipe never waits on list work.
// The query operand (s8 weights 2y - Aq, same K permutation as the byte tiles) lives in tensor memory too
// (A-from-TMEM form of tcgen05.mma: lane = query row, 4 K-elements per 32-bit column), stored once per query
// group with tcgen05.st, so shared-memory bandwidth only carries the document operand.
#pragma once

namespace umma {

constexpr int EPI_WARPS = 8;
constexpr int MMA_WARP = 8;
constexpr int TMA_WARP = 9;
constexpr int THREADS = 320;    // 10 warps: registers are carved per 4 warps, so 12 warps' worth -> 168 per thread
constexpr int STAGE_DOCS = 128;  // N of one MMA
constexpr int ACC_BUFS_MAX = 3;  // 3 x 128 accumulator columns, the query operand behind them (two accumulators for two-part tiles)
constexpr int HIST_BINS = 256;
constexpr int SEED_BINS = 64;     // bins of the sample histogram that seeds the thresholds
constexpr int SEED_STRIDE = EPI_WARPS * 32;  // bin-major shared-memory histograms: counter (copy * 64 + bin) * 256 + thread
__host__ __device__ constexpr int SEED_COPIES(int C) { return C >= 3 ? 2 : 4; }  // 16-bit counters: a copy takes 32 KB
__host__ __device__ constexpr int64_t SEED_MAX_SAMPLE(int C) { return 32768 * SEED_COPIES(C); }  // a 16-bit counter sees at most sample / copies documents
constexpr int TAU_OPEN = -(1 << 30);
constexpr int TAU_NEVER = 1 << 30;     // |acc| <= 512 * 15 * 127 < 2^20, so acc - tau never overflows

struct Params {
    const void *db;            // byte tiles: [ceil(n/128)][C][128 rows x 128 B swizzled] u8 codes
    int64_t n, n_pad, row_offset;
    const unsigned char *qimg; // [nq_pad][128C] s8 weights, K-permuted rows
    const int32_t *qconst;     // [nq_pad] Dq
    const int32_t *tau_init;   // [nq] or nullptr
    int *theta_g;              // [nq] thresholds shared by all CTAs (acc domain, atomicMax), or nullptr
    uint32_t *ghist;           // [nq][HIST_BINS] global histogram of every candidate appended to any list (queue kernel), or nullptr
    const int32_t *theta0;     // [nq] the seeded thresholds the histogram bins are measured from
    int hist_shift;            // bin width = 1 << hist_shift score units
    const int2 *seed_par;      // sample-histogram kernel: per query (origin, reciprocal bin width * 2^32) of its 64 score bins
    int64_t tile_stride;       // sample-histogram kernel: stage i reads byte tile i * tile_stride (the sample is spread over the whole database,
                               // so an ordered or clustered database still gives representative thresholds); n counts the real documents
    uint32_t *seed_hist;       // sample-histogram kernel: [nq][SEED_BINS] counts of sample scores >= origin
    uint64_t *lists;           // [grid][EPI_WARPS][32][cap]
    uint64_t *out;             // [slots * DW][nq][k], KEY_INF pre-filled when slots > 1
    int *list_counts;          // queue kernel, single-wave plans: [grid][queries per CTA] final list lengths -- the lists are not
                               // cut to k and copied out, merge_bounded_kernel reads them where they are; nullptr: emit to `out`
    int64_t nq, stages;
    int groups, k, cap, NS;    // NS = operand stages in shared memory
    int ring_rows;             // queue kernel: rows of a drain warp's ring (32 or 64)
    int n_seg, seg_stages;     // queue kernel: document slices and stages per slice (work items = n_seg x groups)
    int pace;                  // no longer read by the kernels (it selected the roles whose waits were bracketed by clock reads in the
                               // experiment that exposed the yielding wait loop); left in the block because the build without it
                               // ran the main scan 3 % slower -- the code-shape sensitivity described in DESIGN.md section 8, next (1)
    int debug;                 // timing experiments (XFBQ_UMMA_DEBUG): 1 skip operand stores, 2 skip document loads, 4 skip the filter
    unsigned long long *prof;  // optional [grid][8] wait-cycle counters (xfbq_debug_profile), else nullptr
};

using mma::smem_u32;
using mma::mbar_init;
using mma::mbar_arrive;
using mma::mbar_wait;
using mma::Ring;

__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t addr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Shared-memory operand descriptor, K-major, SWIZZLE_128B: rows of 128 bytes, 8-row groups 1024 B apart:
// bits 0-13 start address >> 4 | 16-29 LBO (unused) | 32-45 SBO = 1024 >> 4 | 46-47 version 1 | 61-63 layout 2.
// low word of the descriptor; advancing the start address by `bytes` adds bytes >> 4 (the 14-bit field cannot
// overflow: shared memory ends below 256 KB)
__device__ __forceinline__ uint32_t desc_lo(uint32_t saddr) { return ((saddr >> 4) & 0x3FFFu) | (1u << 16); }
constexpr uint32_t DESC_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
// Instruction descriptor: D = s32 (bits 4-5 = 2), A = signed 8-bit (bits 7-9 = 1: the query weights 2y - Aq), B = UNSIGNED
// 8-bit (bits 10-12 = 0: the document codes, up to 255 for 8-bit codes), both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
#ifndef XFBQ_B_FORMAT
#define XFBQ_B_FORMAT 0u
#endif
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (XFBQ_B_FORMAT << 10) | (static_cast<uint32_t>(STAGE_DOCS >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);

template <bool ACC>
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "mov.b64 db, {%2, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], db, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(IDESC), "n"(ACC ? 1 : 0), "r"(DESC_HI) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint4 &a, const uint4 &b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]),
          "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ bool elect_one() {  // one lane of a converged warp
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
// bar.sync is the .aligned barrier: every thread of a warp must arrive converged.  Role branches end in lane-dependent code
// (`if (lane == 0)`, `if (valid)`), and reconvergence after those is not guaranteed without a warp barrier (synccheck).
// The barrier lives in ONE out-of-line function: every role of a kernel then arrives at the same bar.sync instruction, which
// is what compute-sanitizer's synccheck expects of a CTA-wide barrier (it reports arrivals from different call sites as
// "divergent threads").  Barriers are per work item, not per stage, so the call costs nothing measurable.
__device__ __noinline__ void cta_sync() {
    __syncwarp();
    asm volatile("bar.sync 0;" ::: "memory");
}
__device__ __forceinline__ int max8(const int *v) {
    return max(max(max(v[0], v[1]), v[2]), max(max(max(v[3], v[4]), v[5]), max(v[6], v[7])));
}

// byte offset of (row r, K position kpos) inside a K-major SWIZZLE_128B operand of R rows
__host__ __device__ __forceinline__ uint32_t sw128_offset(int r, int kpos, int R) {
    const int blk = kpos >> 7, kin = kpos & 127;
    return static_cast<uint32_t>(blk * R * 128 + (r >> 3) * 1024 + (r & 7) * 128 + ((((kin >> 4) ^ (r & 7)) & 7) << 4) + (kin & 15));
}

// ------------------------------------------------------------------------------ query operand
// One warp per padded query row.  K position of a dimension = the order in which the producers'
// nibble split emits it: inside a group of 32 dims, word wi = 2e + hi holds bytes j = 0..3 for
// dim = 32g + e + 4hi + 8j.  Rows are plain: the epilogue threads copy theirs into tensor memory.
__global__ void __launch_bounds__(256)
prep_queries_kernel(const uint32_t *__restrict__ q, int64_t nq, int64_t nq_pad, int dim, int wq, int wd, int C, int MT,
                    unsigned char *__restrict__ qimg, int32_t *__restrict__ qconst) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= nq_pad) return;
    const int W = 4 * ((dim + 127) >> 7);  // words per plane of the query layout (C may be padded to an even chunk count)
    const int Aq = (1 << wq) - 1, Ad = (1 << wd) - 1;
    unsigned char *img = qimg + row * (static_cast<int64_t>(C) * 128);
    (void)MT;
    int sy = 0;
    for (int ow = lane; ow < 32 * C; ow += 32) {
        const int g = ow >> 3, wi = ow & 7, e = wi >> 1, hi = wi & 1;
        uint32_t packed = 0;
        if (row < nq) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int d = 32 * g + e + 4 * hi + 8 * j;
                const int word = d >> 5, bit = d & 31;
                int y = 0, w = 0;
                if (d < dim) {
                    for (int jq = 0; jq < wq; ++jq) y |= static_cast<int>((q[(row * wq + jq) * W + word] >> bit) & 1u) << jq;
                    w = 2 * y - Aq; sy += y;
                }
                packed |= (static_cast<uint32_t>(w) & 0xFFu) << (8 * j);
            }
        }
        *reinterpret_cast<uint32_t *>(img + 4 * ow) = packed;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sy += __shfl_xor_sync(0xffffffffu, sy, o);
    if (lane == 0) qconst[row] = (row < nq) ? Ad * sy : 0;
}

struct SmemLayout {
    uint32_t a_off, b_off, hist_off, bar_off, total;
};
__host__ __device__ inline SmemLayout smem_layout(int C, int MT, int NS, bool seed_hist = false) {
    SmemLayout L;
    uint32_t off = 0;
    L.a_off = off; (void)MT;
    L.b_off = off; off += static_cast<uint32_t>(NS) * STAGE_DOCS * 128 * C;
    L.hist_off = off; off += seed_hist ? SEED_COPIES(C) * SEED_STRIDE * SEED_BINS * 2 : EPI_WARPS * 256 * 4;
    L.bar_off = off; off += (2 * NS + 2 * ACC_BUFS_MAX) * 8 + 16;
    L.total = off + 1024;  // slack for the manual 1024-byte alignment of the operand area
    return L;
}

// nibble layout -> byte tiles; one thread per (document, group of 32 dims).  A group's nibble word e holds in
// nibble m the code of dim 4m + e: even / odd nibbles split into words (e, lo), (e, hi) -> K positions
// 32g + 8e + 4hi + j for dim 32g + e + 4hi + 8j (prep_queries_kernel applies the same permutation).
__global__ void __launch_bounds__(256)
nibbles_to_tiles_kernel(const uint4 *__restrict__ nib, int64_t n_pad, int64_t n_tiles, int C, unsigned char *__restrict__ tiles) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int G = 4 * C;
    if (e >= n_tiles * STAGE_DOCS * G) return;
    const int64_t doc = e / G;
    const int g = static_cast<int>(e - doc * G);
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (doc < n_pad) w = nib[doc * G + g];
    const int64_t tile = doc / STAGE_DOCS;
    const int r = static_cast<int>(doc - tile * STAGE_DOCS);
    const int kb = g >> 2, gg = g & 3;
    unsigned char *rowp = tiles + tile * (static_cast<int64_t>(STAGE_DOCS) * 128 * C) + kb * (STAGE_DOCS * 128) + (r >> 3) * 1024 + (r & 7) * 128;
    *reinterpret_cast<uint4 *>(rowp + (((2 * gg) ^ (r & 7)) << 4)) =
        make_uint4(w.x & 0x0F0F0F0Fu, (w.x >> 4) & 0x0F0F0F0Fu, w.y & 0x0F0F0F0Fu, (w.y >> 4) & 0x0F0F0F0Fu);
    *reinterpret_cast<uint4 *>(rowp + (((2 * gg + 1) ^ (r & 7)) << 4)) =
        make_uint4(w.z & 0x0F0F0F0Fu, (w.z >> 4) & 0x0F0F0F0Fu, w.w & 0x0F0F0F0Fu, (w.w >> 4) & 0x0F0F0F0Fu);
}

// bundle layout (bit planes) -> byte tiles directly, any code width 1..8; one thread per (document, group of 32 dims).
// Plane i's 32-bit word of the group holds dim d in bit d, so ((P_i >> (e + 4 hi)) & 0x01010101) << i places bit i of the
// codes of dims e + 4 hi + {0, 8, 16, 24} into bytes j = 0..3 of output word (e, hi): the same K order as above.
__global__ void __launch_bounds__(256)
planes_to_tiles_kernel(const uint32_t *__restrict__ db, int64_t n_pad, int64_t n_tiles, int wd, int CP, int C, unsigned char *__restrict__ tiles) {
    // CP = chunks of the bundle layout (ceil(dim / 128)), C >= CP = chunks of a tile (padded to an even count above 4)
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int G = 4 * C;
    if (e >= n_tiles * STAGE_DOCS * G) return;
    const int64_t doc = e / G;
    const int g = static_cast<int>(e - doc * G);
    uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // w[2 e + hi]
    if (doc < n_pad && (g >> 2) < CP) {
        const int64_t b = doc >> 5;
        const int l = static_cast<int>(doc & 31), c = g >> 2;
        for (int i = 0; i < wd; ++i) {
            const uint32_t pw = __ldg(db + ((((b * wd + i) * CP + c) * 32 + l) << 2) + (g & 3));
#pragma unroll
            for (int x = 0; x < 8; ++x) w[x] |= ((pw >> ((x >> 1) + 4 * (x & 1))) & 0x01010101u) << i;
        }
    }
    const int64_t tile = doc / STAGE_DOCS;
    const int r = static_cast<int>(doc - tile * STAGE_DOCS);
    const int kb = g >> 2, gg = g & 3;
    unsigned char *rowp = tiles + tile * (static_cast<int64_t>(STAGE_DOCS) * 128 * C) + kb * (STAGE_DOCS * 128) + (r >> 3) * 1024 + (r & 7) * 128;
    *reinterpret_cast<uint4 *>(rowp + (((2 * gg) ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4 *>(rowp + (((2 * gg + 1) ^ (r & 7)) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
}

// byte tiles -> bundle layout (bit planes): the inverse of planes_to_tiles_kernel, one thread per (document, group of 32 dims).
// Lets a server that only answers large batches keep the tiles alone and rebuild the packed codes when something needs them.
__global__ void __launch_bounds__(256)
tiles_to_planes_kernel(const unsigned char *__restrict__ tiles, int64_t n_pad, int wd, int CP, int C, uint32_t *__restrict__ db) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int G = 4 * CP;  // groups of the bundle layout; the tile may hold padded chunks beyond them
    if (e >= n_pad * G) return;
    const int64_t doc = e / G;
    const int g = static_cast<int>(e - doc * G);
    const int64_t tile = doc / STAGE_DOCS;
    const int r = static_cast<int>(doc - tile * STAGE_DOCS);
    const int kb = g >> 2, gg = g & 3;
    const unsigned char *rowp = tiles + tile * (static_cast<int64_t>(STAGE_DOCS) * 128 * C) + kb * (STAGE_DOCS * 128) + (r >> 3) * 1024 + (r & 7) * 128;
    const uint4 lo = *reinterpret_cast<const uint4 *>(rowp + (((2 * gg) ^ (r & 7)) << 4));
    const uint4 hi = *reinterpret_cast<const uint4 *>(rowp + (((2 * gg + 1) ^ (r & 7)) << 4));
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};  // w[2 e + hi]: bytes j = codes of dims e + 4 hi + 8 j
    const int64_t b = doc >> 5;
    const int l = static_cast<int>(doc & 31);
    for (int i = 0; i < wd; ++i) {
        uint32_t pw = 0u;
#pragma unroll
        for (int x = 0; x < 8; ++x) pw |= ((w[x] >> i) & 0x01010101u) << ((x >> 1) + 4 * (x & 1));
        db[((((b * wd + i) * CP + kb) * 32 + l) << 2) + gg] = pw;
    }
}

// mbarrier wait (every lane polls: measured far faster than one polling lane + warp barrier) that adds the
// cycles spent waiting to `acc` when profiling is on
__device__ __forceinline__ void mbar_wait_prof(uint64_t *bar, uint32_t parity, bool prof, long long &acc) {
    if (!prof) { mbar_wait(bar, parity); return; }
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
}

// mbarrier wait with the retry loop inside the asm block.  Around a C++ loop the compiler places a YIELD in front of
// every try_wait, the first one included: the warp hands its issue slot to the other warps of its scheduler even when
// the barrier has already completed.  For the MMA issuer (one warp, on the critical path of the tensor pipe, sharing
// a scheduler with three busy drain warps) that cost 5 % of the scan (found through the profiling counters: their
// clock reads happened to move the first try_wait out of the yielding loop).
__device__ __forceinline__ void mbar_wait_tight(uint64_t *bar, uint32_t parity) {
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

// v[j] for a warp-uniform j without dynamic register indexing (a jump table of 32 moves)
__device__ __forceinline__ int pick32(const int (&v)[32], int j) {
    int r = v[0];
    switch (j) {
#define XFBQ_PICK(J) case J: r = v[J]; break;
        XFBQ_PICK(1) XFBQ_PICK(2) XFBQ_PICK(3) XFBQ_PICK(4) XFBQ_PICK(5) XFBQ_PICK(6) XFBQ_PICK(7) XFBQ_PICK(8)
        XFBQ_PICK(9) XFBQ_PICK(10) XFBQ_PICK(11) XFBQ_PICK(12) XFBQ_PICK(13) XFBQ_PICK(14) XFBQ_PICK(15) XFBQ_PICK(16)
        XFBQ_PICK(17) XFBQ_PICK(18) XFBQ_PICK(19) XFBQ_PICK(20) XFBQ_PICK(21) XFBQ_PICK(22) XFBQ_PICK(23) XFBQ_PICK(24)
        XFBQ_PICK(25) XFBQ_PICK(26) XFBQ_PICK(27) XFBQ_PICK(28) XFBQ_PICK(29) XFBQ_PICK(30) XFBQ_PICK(31)
#undef XFBQ_PICK
        default: break;
    }
    return r;
}

// Warp-level radix select for short lists (cnt <= 32 * KPL): same contract as mma::select_row (keeps exactly
// the k smallest of the cnt > k unique keys at the front of the row, returns the k-th), but the keys are
// read from L2 once and every pass works on registers, so a compaction costs one L2 round trip instead of
// one per pass.
template <int KPL>
__device__ __noinline__ uint64_t select_small(uint64_t *row, int cnt, int k, int *hist, int lane) {
    __syncwarp();
    uint64_t key[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) key[i] = (i * 32 + lane < cnt) ? __ldcg(row + i * 32 + lane) : KEY_INF;
    const uint64_t first = mma::shfl_u64(key[0], 0);
    uint64_t diff = 0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) if (i * 32 + lane < cnt) diff |= key[i] ^ first;
    {
        const uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(diff));
        const uint32_t hi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(diff >> 32));
        diff = (static_cast<uint64_t>(hi) << 32) | lo;
    }
    int shift = ((63 - __clzll(static_cast<long long>(diff | 1ull))) >> 3) << 3;  // byte holding the top differing bit
    uint64_t hi_mask = shift + 8 >= 64 ? 0ull : ~((1ull << (shift + 8)) - 1ull);    // bits common to all keys
    uint64_t prefix = first & hi_mask;
    int want = k;
    while (true) {
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[8 * lane + b] = 0;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < KPL; ++i)
            if (i * 32 + lane < cnt && (key[i] & hi_mask) == prefix) atomicAdd(&hist[static_cast<int>(key[i] >> shift) & 255], 1);
        __syncwarp();
        int h[8], sum = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) { h[e] = hist[8 * lane + e]; sum += h[e]; }
        int inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const int exc = inc - sum;
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
    uint64_t kth = 0;
    int out = 0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
        const bool keep = i * 32 + lane < cnt && (key[i] & hi_mask) <= prefix;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            row[out + __popc(m & ((1u << lane) - 1u))] = key[i];
            kth = key[i] > kth ? key[i] : kth;
        }
        out += __popc(m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t other = mma::shfl_u64(kth, lane ^ o);
        kth = other > kth ? other : kth;
    }
    __syncwarp();
    return kth;
}
__device__ __forceinline__ uint64_t select_any(uint64_t *row, int cnt, int k, int *hist, int lane) {
    if (cnt <= 256) return select_small<8>(row, cnt, k, hist, lane);
    return mma::select_row(row, cnt, k, hist, lane);
}

// A CTA's share of the linearised (group, stage) work, cut into segments of one query group each.
struct Segments {
    int64_t lin, lin_end, T;
    int gr, sd0, cnt;
    __device__ __forceinline__ bool next() {
        if (lin >= lin_end) return false;
        gr = static_cast<int>(lin / T);
        sd0 = static_cast<int>(lin - static_cast<int64_t>(gr) * T);
        int64_t left = lin_end - lin;
        if (left > T - sd0) left = T - sd0;
        cnt = static_cast<int>(left);
        lin += left;
        return true;
    }
};

// Work items of the queue kernel: the documents are cut into `n_seg` slices, item w = (slice w / groups,
// query group w % groups), and CTA c takes items c, c + gridDim.x, ...  Items that run at the same time are
// then the query groups of the same few document slices, walking them roughly in step: every byte tile is
// fetched from HBM about once and served to the other ~40 CTAs by the L2 (with the linearised ranges of the
// kernel above all 148 CTAs stream different tiles: 84 GB of DRAM reads per 10k-query launch, measured).
struct Items {
    int64_t w, w_end, stride;
    int groups, seg_stages, T;
    int gr, sd0, cnt, part;
    __device__ __forceinline__ bool next() {
        if (w >= w_end) return false;
        part = static_cast<int>(w / groups);
        gr = static_cast<int>(w - static_cast<int64_t>(part) * groups);
        sd0 = part * seg_stages;
        cnt = T - sd0 < seg_stages ? T - sd0 : seg_stages;
        w += stride;
        return true;
    }
};

// SEED = true turns the epilogue into a counter: no lists, no thresholds -- every sample score at or above the
// query's bin origin bumps one of 64 bins (a shared-memory row owned by the thread, flushed to the global
// histogram of the query when the CTA leaves the group).  seed_bounds_kernel then reads a valid threshold off
// the histogram: "the bins >= b hold k real documents".  Seeding by list maintenance from open thresholds cost
// 2.2 ms per 10k queries, two thirds of it in list compactions.
// KP = 2: documents of 513..1024 dims as tiles of two K parts (C chunks each, streamed as two operand stages that
// accumulate into one accumulator); two accumulators, one query tile.
template <int C, int MT, bool SEED = false, int KP = 1>
__global__ void __launch_bounds__(THREADS, 1) scan_kernel(const Params p) {
    constexpr int B_STAGE = STAGE_DOCS * 128 * C;     // one document stage = one byte tile
    constexpr int KSTEPS = 4 * C;                     // K = 32 per MMA
    constexpr int COLS = MT == 2 ? 128 : 64;          // accumulator columns an epilogue warp drains
    constexpr int EPI_PER_BUF = MT == 2 ? 4 : 8;      // epilogue warps reading one accumulator
    constexpr int A_COLS = 32 * C * KP;               // tensor-memory columns of one 128-query operand tile (all K parts)
    constexpr int AB = KP == 1 ? ACC_BUFS_MAX : 2;    // accumulators: the operand of a two-part tile takes up to 256 columns
    constexpr int ACOL0 = AB * STAGE_DOCS;
    static_assert(KP == 1 || MT == 1, "two-part tiles leave room for one query tile");                    // tensor-memory columns of one 128-query operand tile
    extern __shared__ unsigned char smem_unaligned[];
    const uint32_t pad = (1024u - (smem_u32(smem_unaligned) & 1023u)) & 1023u;
    unsigned char *smem = smem_unaligned + pad;
    const int NS = p.NS;
    const SmemLayout L = smem_layout(C, MT, NS, SEED);
    unsigned char *sB = smem + L.b_off;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bar_off);
    uint64_t *b_full = bars, *b_empty = bars + NS, *acc_full = bars + 2 * NS, *acc_empty = bars + 2 * NS + AB;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NS + 2 * AB);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const int64_t T = p.stages;
    const int64_t W = static_cast<int64_t>(p.groups) * T;
    const int64_t G = gridDim.x;
    Segments sg{static_cast<int64_t>(blockIdx.x) * W / G, (static_cast<int64_t>(blockIdx.x) + 1) * W / G, T, 0, 0, 0};

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
        for (int i = 0; i < AB; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], EPI_PER_BUF); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    fence_before();
    cta_sync();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // Every role runs the same segment loop:  [epilogue: store the group's query operand to tensor memory]
    // | barrier | role work | barrier (every MMA that read the operand is done: the epilogue has consumed
    // its result).
    uint32_t s_run = 0;  // stages this CTA has processed so far (drives every ring cursor)
    const bool prof = p.prof != nullptr;
    long long w0 = 0, w1 = 0;
    int w2 = 0;
    const long long t_begin = prof ? clock64() : 0;

    if (warp < EPI_WARPS) {
        // ================================ epilogue ================================
        const int q4 = warp & 3, idx = warp >> 2;
        const int mt = MT == 2 ? idx : 0;
        const int col0 = MT == 2 ? 0 : idx * COLS;
        uint64_t *warp_lists = p.lists + (static_cast<int64_t>(blockIdx.x) * EPI_WARPS + warp) * 32 * static_cast<int64_t>(p.cap);
        uint64_t *my_list = warp_lists + static_cast<int64_t>(lane) * p.cap;
        int *hist = reinterpret_cast<int *>(smem + L.hist_off) + warp * 256;
        const uint32_t n_docs = static_cast<uint32_t>(p.n);
        const uint32_t id_off = static_cast<uint32_t>(p.row_offset);  // row ids fit 32 bits (checked on the host)
        const int cap = p.cap, k = p.k;
        while (sg.next()) {
            const int64_t q0 = (static_cast<int64_t>(sg.gr) * MT + mt) * 128 + q4 * 32;  // first query row of this warp
            const int64_t myq = q0 + lane;
            if (MT == 2 || idx == 0) {  // this thread's query row -> lane (32 q4 + lane), columns of tile mt
                const uint4 *src = reinterpret_cast<const uint4 *>(p.qimg + myq * (128 * C * KP));
                const uint32_t ta = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + ACOL0 + mt * A_COLS;
#pragma unroll
                for (int c = 0; c < A_COLS / 8; ++c) tmem_st8(ta + c * 8, __ldg(src + 2 * c), __ldg(src + 2 * c + 1));
                tmem_st_wait();
            }
            fence_before();
            cta_sync();
            const bool valid = myq < p.nq;
            if constexpr (SEED) {
                // Counting epilogue.  This thread's bins are 16-bit counters of its own in shared memory, bin-major
                // (row (copy * 64 + bin) of 256 counters, a thread's slot chosen so that a warp never conflicts), in SEED_COPIES
                // copies: column j updates copy j % COPIES, so COPIES read-modify-writes are in flight at a time
                // (plain LDS/ADD/STS: shared-memory atomics -- and the divergent branches ptxas wraps around
                // predicated ones -- bounded the first version at 11k cycles per stage).
                constexpr int COPIES = SEED_COPIES(C);
                // 16-bit counter of (bin row, thread): word (warp / 2) * 32 + lane, half warp & 1 -- a warp's 32 accesses fall in
                // 32 different banks whatever their bins (thread-linear halves put lanes 2i, 2i + 1 in one bank: 2-way conflicts)
                const uint32_t bins_s = smem_u32(smem + L.hist_off) + ((warp >> 1) * 32 + lane) * 4 + (warp & 1) * 2;
                for (int b = 0; b < COPIES * SEED_BINS; ++b)
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(bins_s + b * (SEED_STRIDE * 2)), "h"(static_cast<unsigned short>(0)) : "memory");
                // frame of this query: bin(v) = clamp(floor((v - origin) / width) + 1, 0, 63) computed as a signed
                // multiply-high; bin 0 collects everything below the origin, so every score is one unconditional
                // read-modify-write (sampled tiles hold real documents only: the host keeps them off the last tile)
                const int2 par = valid ? p.seed_par[myq] : make_int2(0, 0);
                const int c2 = par.x;   // 2 * (origin - width)
                const int m31 = par.y;  // ceil(2^31 / width)
                const uint32_t u0 = s_run * MT + mt;
                Ring ac{static_cast<int>(u0 % AB), (u0 / AB) & 1u};
                for (int i = 0; i < sg.cnt; ++i) {
                    const uint32_t buf = ac.idx;
                    mbar_wait_prof(&acc_full[buf], ac.phase, prof, w0);
                    fence_after();
                    const uint32_t taddr = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + buf * STAGE_DOCS + col0;
                    int v[COLS / 32][32];
#pragma unroll
                    for (int c = 0; c < COLS / 32; ++c) tmem_ld32(taddr + c * 32, v[c]);
                    tmem_ld_wait();
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&acc_empty[buf]);
#pragma unroll
                    for (int c = 0; c < COLS / 32; ++c)
#pragma unroll
                        for (int j0 = 0; j0 < 32; j0 += COPIES) {
                            uint32_t addr[COPIES];
                            unsigned short cur[COPIES];
#pragma unroll
                            for (int u = 0; u < COPIES; ++u) {
                                const int h = __mulhi(2 * v[c][j0 + u] - c2, m31);
                                const int bin = min(max(h, 0), SEED_BINS - 1);
                                addr[u] = bins_s + u * (SEED_BINS * SEED_STRIDE * 2) + bin * (SEED_STRIDE * 2);
                            }
#pragma unroll
                            for (int u = 0; u < COPIES; ++u) asm volatile("ld.shared.u16 %0, [%1];" : "=h"(cur[u]) : "r"(addr[u]) : "memory");
#pragma unroll
                            for (int u = 0; u < COPIES; ++u)
                                asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr[u]), "h"(static_cast<unsigned short>(cur[u] + 1)) : "memory");
                        }
#pragma unroll
                    for (int a = 0; a < MT; ++a) ac.advance(AB);
                }
                if (valid)
                    for (int b = 1; b < SEED_BINS; ++b) {  // bin 0 (below the origin) proves nothing
                        uint32_t c = 0;
#pragma unroll
                        for (int u = 0; u < COPIES; ++u) {
                            unsigned short x;
                            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(x) : "r"(bins_s + (u * SEED_BINS + b) * (SEED_STRIDE * 2)) : "memory");
                            c += x;
                        }
                        if (c) atomicAdd(p.seed_hist + myq * SEED_BINS + b, c);
                    }
                s_run += static_cast<uint32_t>(sg.cnt);
                cta_sync();
                continue;
            }
            const int dq = valid ? p.qconst[myq] : 0;
            int theta = valid ? (p.tau_init ? max(TAU_OPEN, p.tau_init[myq]) : TAU_OPEN) : TAU_NEVER;
            int cnt = 0;

            // 32 scores of this thread's query row: 3-input max tree, one compare, one vote.  On a hit (rare
            // once thresholds have tightened) the warp builds per-lane hit masks from sign bits.  A lane with
            // exactly one hit -- the common case -- knows the score already (it is the row maximum) and the
            // column from the mask; only lanes with several hits walk their columns (jump-table pick).
            auto filter = [&](const int (&v)[32], uint32_t doc0) {
                const int g0 = max8(v), g1 = max8(v + 8), g2 = max8(v + 16), g3 = max8(v + 24);
                const int m = max(max(g0, g1), max(g2, g3));
                if (__any_sync(0xffffffffu, m >= theta)) {
                    ++w1;
                    const int gm[4] = {g0, g1, g2, g3};
                    uint32_t hits = 0;
#pragma unroll
                    for (int qg = 0; qg < 4; ++qg)
                        if (__any_sync(0xffffffffu, gm[qg] >= theta)) {
                            uint32_t below = 0;  // bit j: v[8 qg + j] < theta
#pragma unroll
                            for (int j = 7; j >= 0; --j) below = __funnelshift_l(static_cast<uint32_t>(v[8 * qg + j] - theta), below, 1);
                            hits |= (~below & 0xFFu) << (8 * qg);
                        }
                    const bool single = (hits & (hits - 1)) == 0;
                    if (hits && single) {
                        const uint32_t doc = doc0 + (__ffs(hits) - 1);
                        if (doc < n_docs) {
                            my_list[cnt] = (static_cast<uint64_t>(static_cast<uint32_t>(dq - m)) << 32) | (id_off + doc);
                            ++cnt;
                        }
                    }
                    uint32_t cols = __reduce_or_sync(0xffffffffu, single ? 0u : hits);
                    if (__popc(cols) > 6) {
                        // dense hits (open or young thresholds: the sample scans): one predicated pass over the
                        // 32 columns beats walking their union one jump-table pick at a time
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (!single && ((hits >> j) & 1u) && doc0 + j < n_docs) {
                                my_list[cnt] = (static_cast<uint64_t>(static_cast<uint32_t>(dq - v[j])) << 32) | (id_off + doc0 + j);
                                ++cnt;
                            }
                    } else {
                        while (cols) {
                            const int j = __ffs(cols) - 1;
                            cols &= cols - 1;
                            const int val = pick32(v, j);
                            if (!single && ((hits >> j) & 1u) && doc0 + j < n_docs) {
                                my_list[cnt] = (static_cast<uint64_t>(static_cast<uint32_t>(dq - val)) << 32) | (id_off + doc0 + j);
                                ++cnt;
                            }
                        }
                    }
                    __syncwarp();
                    unsigned need = __ballot_sync(0xffffffffu, cnt > cap - 32);
                    if (need) {
                        w2 += __popc(need);
                        do {  // a list that the next 32 documents could overflow: keep its k best
                            const int ql = __ffs(need) - 1;
                            need &= need - 1;
                            const int c = __shfl_sync(0xffffffffu, cnt, ql);
                            const uint64_t kth = select_any(warp_lists + static_cast<int64_t>(ql) * cap, c, k, hist, lane);
                            if (lane == ql) {
                                cnt = k;
                                theta = dq - static_cast<int>(kth >> 32);
                                if (p.theta_g) atomicMax(p.theta_g + myq, theta);  // every CTA scanning this query tightens with us
                            }
                        } while (need);
                    }
                }
            };

            const uint32_t u0 = s_run * MT + mt;
            Ring ac{static_cast<int>(u0 % AB), (u0 / AB) & 1u};
            // thresholds other CTAs found for this query: fetched four stages ahead of their use, so the L2 round
            // trip never sits on a stage's critical path
            const bool fetch_shared = p.theta_g && valid;
            int shared_next = TAU_OPEN;
            for (int i = 0; i < sg.cnt; ++i) {
                const uint32_t buf = ac.idx;
                int shared_theta = TAU_OPEN;
                if ((i & 3) == 0) {
                    shared_theta = shared_next;
                    if (fetch_shared) shared_next = __ldcg(p.theta_g + myq);
                }
                mbar_wait_prof(&acc_full[buf], ac.phase, prof, w0);
                fence_after();
                const uint32_t taddr = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + buf * STAGE_DOCS + col0;
                const uint32_t doc0 = static_cast<uint32_t>(sg.sd0 + i) * STAGE_DOCS + col0;
                // the whole accumulator slice goes to registers first, so the buffer returns to the issuer after
                // one tensor-memory read time instead of after the filter: it is on the MMA pipe's critical path
                int v[COLS / 32][32];
                if (!(p.debug & 4)) {
#pragma unroll
                    for (int c = 0; c < COLS / 32; ++c) tmem_ld32(taddr + c * 32, v[c]);
                    tmem_ld_wait();
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
                theta = max(theta, shared_theta);
                if (!(p.debug & 4)) {
#pragma unroll
                    for (int c = 0; c < COLS / 32; ++c) filter(v[c], doc0 + c * 32);
                }
#pragma unroll
                for (int a = 0; a < MT; ++a) ac.advance(AB);
            }
            // ---- emit: every query row of this warp, its <= k best keys (unsorted), KEY_INF padded
            {
                int64_t c_first = (static_cast<int64_t>(sg.gr) * T * G) / W;
                while (c_first > 0 && c_first * W / G > static_cast<int64_t>(sg.gr) * T) --c_first;
                while ((c_first + 1) * W / G <= static_cast<int64_t>(sg.gr) * T) ++c_first;
                const int64_t part = (static_cast<int64_t>(blockIdx.x) - c_first) * (MT == 2 ? 1 : 2) + (MT == 2 ? 0 : idx);
                __syncwarp();
                for (int ql = 0; ql < 32; ++ql) {
                    const int64_t qq = q0 + ql;
                    if (qq >= p.nq) break;
                    int c = __shfl_sync(0xffffffffu, cnt, ql);
                    uint64_t *row = warp_lists + static_cast<int64_t>(ql) * cap;
                    if (c > k) { select_any(row, c, k, hist, lane); c = k; }
                    __syncwarp();
                    uint64_t *dst = p.out + (part * p.nq + qq) * k;
                    for (int e = lane; e < k; e += 32) dst[e] = e < c ? __ldcg(row + e) : KEY_INF;
                }
                __syncwarp();
            }
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
        if (prof && threadIdx.x == 0) {
            unsigned long long *o = p.prof + blockIdx.x * 8, *x = p.prof + gridDim.x * 8 + blockIdx.x * 4;
            o[0] = w0; o[1] = w1; o[6] = clock64() - t_begin; o[7] = s_run;
            x[0] = 0; x[1] = 0; x[2] = w2;
        }
    } else if (warp == MMA_WARP) {
        // ================================ MMA issuer ================================
        const uint32_t b_lo0 = desc_lo(smem_u32(sB));
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // warp-uniform by construction
        while (sg.next()) {
            cta_sync();
            fence_after();  // the query operand stored by the epilogue warps is in tensor memory
            Ring rb{static_cast<int>((s_run * KP) % NS), ((s_run * KP) / NS) & 1u};
            const uint32_t u0 = s_run * MT;
            Ring ac{static_cast<int>(u0 % AB), ((u0 / AB) & 1u) ^ 1u};  // "empty" waits: completed phase first
            for (int i = 0; i < sg.cnt; ++i) {  // the whole warp walks the pipeline, one elected lane issues
                if constexpr (KP > 1) {  // one accumulator per tile, fed by KP operand stages
                    const uint32_t buf = ac.idx;
                    mbar_wait_prof(&acc_empty[buf], ac.phase, prof, w1);
                    fence_after();
#pragma unroll
                    for (int part = 0; part < KP; ++part) {
                        mbar_wait_prof(&b_full[rb.idx], rb.phase, prof, w0);
                        fence_after();
                        const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(rb.idx) * (B_STAGE >> 4);
                        if (elect_one()) {
                            const uint32_t d = tm + buf * STAGE_DOCS;
#pragma unroll
                            for (int ks = 0; ks < KSTEPS; ++ks) {
                                const uint32_t ta = tm + ACOL0 + (part * KSTEPS + ks) * 8;
                                const uint32_t bo = ((ks >> 2) * (STAGE_DOCS * 128) + (ks & 3) * 32) >> 4;
                                if (part == 0 && ks == 0) umma_i8<false>(d, ta, b_lo + bo);
                                else umma_i8<true>(d, ta, b_lo + bo);
                            }
                            umma_commit(&b_empty[rb.idx]);
                            if (part == KP - 1) umma_commit(&acc_full[buf]);
                        }
                        __syncwarp();
                        rb.advance(NS);
                    }
                    ac.advance(AB);
                    continue;
                }
                mbar_wait_prof(&b_full[rb.idx], rb.phase, prof, w0);
                fence_after();
                const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(rb.idx) * (B_STAGE >> 4);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const uint32_t buf = ac.idx;
                    mbar_wait_prof(&acc_empty[buf], ac.phase, prof, w1);
                    fence_after();
                    if (elect_one()) {
                        const uint32_t d = tm + buf * STAGE_DOCS;
#pragma unroll
                        for (int ks = 0; ks < KSTEPS; ++ks) {
                            const uint32_t ta = tm + ACOL0 + mt * A_COLS + ks * 8;  // K = 32 signed bytes = 8 columns
                            const uint32_t bo = ((ks >> 2) * (STAGE_DOCS * 128) + (ks & 3) * 32) >> 4;
                            if (ks == 0) umma_i8<false>(d, ta, b_lo + bo);
                            else umma_i8<true>(d, ta, b_lo + bo);
                        }
                        umma_commit(&acc_full[buf]);
                    }
                    __syncwarp();
                    ac.advance(AB);
                }
                if (elect_one()) umma_commit(&b_empty[rb.idx]);
                __syncwarp();
                rb.advance(NS);
            }
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
        if (prof && lane == 0) { p.prof[blockIdx.x * 8 + 2] = w0; p.prof[blockIdx.x * 8 + 3] = w1; }
    } else {
        // ================================ loader ================================
        const unsigned char *db = reinterpret_cast<const unsigned char *>(p.db);
        while (sg.next()) {
            cta_sync();
            if (lane == 0) {
                Ring rb{static_cast<int>((s_run * KP) % NS), (((s_run * KP) / NS) & 1u) ^ 1u};  // "empty" waits start on the completed phase
                for (int i = 0; i < sg.cnt; ++i) {
#pragma unroll
                    for (int part = 0; part < KP; ++part) {
                        mbar_wait_prof(&b_empty[rb.idx], rb.phase, prof, w0);
                        mma::mbar_arrive_expect_tx(&b_full[rb.idx], B_STAGE);
                        mma::tma_bulk_g2s(sB + static_cast<size_t>(rb.idx) * B_STAGE,
                                          db + (static_cast<int64_t>(sg.sd0 + i) * (SEED ? p.tile_stride : 1) * KP + part) * B_STAGE, B_STAGE, &b_full[rb.idx]);
                        rb.advance(NS);
                    }
                }
            }
            __syncwarp();
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
        if (prof && lane == 0) { p.prof[blockIdx.x * 8 + 4] = w0; p.prof[blockIdx.x * 8 + 5] = 0; }
    }
    fence_before();
    cta_sync();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------------------ threshold seeding by counting
// seed_stats_kernel: one block of 128 threads per query scores 128 documents spread over the sample (row i of
// every (tiles/128)-th sampled byte tile) with dp4a, and turns mean and deviation of those scores into the query's bin
// frame: origin = mean + (z - 3) sigma, 64 bins of sigma/16, where z is the normal quantile of the k-th best of
// the sample.  The frame only has to bracket the k-th best sample score; any frame gives a VALID threshold
// (bins count real documents), a poor one a loose or open threshold.
__device__ __forceinline__ int dp4a_su(uint32_t a_s8x4, uint32_t b_u8x4, int c) {
    int d;
    asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_s8x4), "r"(b_u8x4), "r"(c));
    return d;
}
__global__ void __launch_bounds__(128) seed_stats_kernel(const unsigned char *__restrict__ tiles, const unsigned char *__restrict__ qimg,
                                                         int64_t nq, int C, int64_t sample_tiles, int64_t tile_stride, float z, float below, int2 *__restrict__ par,
                                                         uint32_t *__restrict__ seed_hist) {
    const int64_t q = blockIdx.x;
    const int r = threadIdx.x;
    if (r < SEED_BINS) seed_hist[q * SEED_BINS + r] = 0u;  // the counting scan that follows adds to it (one stream operation less than a memset)
    const int64_t t = (static_cast<int64_t>(r) * sample_tiles / 128) * tile_stride;
    const unsigned char *tile = tiles + t * (static_cast<int64_t>(STAGE_DOCS) * 128 * C);
    const uint4 *qrow = reinterpret_cast<const uint4 *>(qimg + q * (128 * C));
    int acc = 0;
    for (int u = 0; u < 8 * C; ++u) {
        const uint4 a = __ldg(qrow + u);
        const uint4 b = __ldg(reinterpret_cast<const uint4 *>(tile + sw128_offset(r, u * 16, STAGE_DOCS)));
        acc = dp4a_su(a.x, b.x, acc);  // signed query weights x unsigned document codes
        acc = dp4a_su(a.y, b.y, acc);
        acc = dp4a_su(a.z, b.z, acc);
        acc = dp4a_su(a.w, b.w, acc);
    }
    __shared__ float s_sum[4], s_sq[4];
    float s = static_cast<float>(acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((r & 31) == 0) s_sum[r >> 5] = s;
    __syncthreads();
    const float mean = (s_sum[0] + s_sum[1] + s_sum[2] + s_sum[3]) * (1.0f / 128.0f);
    const float dv = static_cast<float>(acc) - mean;
    float sq = dv * dv;
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((r & 31) == 0) s_sq[r >> 5] = sq;
    __syncthreads();
    if (r == 0) {
        const float sigma = sqrtf((s_sq[0] + s_sq[1] + s_sq[2] + s_sq[3]) * (1.0f / 127.0f));
        const float width = fmaxf(2.0f, rintf(sigma * (1.0f / 16.0f)));
        const int origin = static_cast<int>(floorf(mean + (z - below) * sigma));
        const int w = static_cast<int>(width);
        par[q] = make_int2(2 * (origin - w), static_cast<int>((0x80000000ll + w - 1) / w));
    }
}

// seed_bounds_kernel: one warp per query reads the threshold off the sample histogram: the largest bin b whose
// suffix count reaches k proves that k real documents score at least origin + d_b, d_b = the smallest offset
// that maps to bin b.  TAU_OPEN when the frame missed (fewer than k sample scores at or above the origin).
__global__ void __launch_bounds__(256) seed_bounds_kernel(const uint32_t *__restrict__ hist, const int2 *__restrict__ par,
                                                          int64_t nq, int k, int32_t *__restrict__ tau,
                                                          int32_t *__restrict__ theta0, uint32_t *__restrict__ ghist) {
    const int64_t q = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= nq) return;
    if (ghist) {  // the main scan's candidate histogram of this query starts empty (instead of a memset + a copy of the thresholds)
        uint4 *row = reinterpret_cast<uint4 *>(ghist + q * HIST_BINS) + 2 * lane;
        row[0] = make_uint4(0u, 0u, 0u, 0u);
        row[1] = make_uint4(0u, 0u, 0u, 0u);
    }
    const uint2 c = *reinterpret_cast<const uint2 *>(hist + q * SEED_BINS + 2 * lane);  // bins 2 lane, 2 lane + 1
    const uint32_t s = c.x + c.y;
    uint32_t suf = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += v;
    }
    const uint32_t kk = static_cast<uint32_t>(k);
    const bool mine = suf >= kk && suf - s < kk;
    const int b = (suf - s + c.y >= kk) ? 2 * lane + 1 : 2 * lane;
    const unsigned m = __ballot_sync(0xffffffffu, mine);
    const int bb = __shfl_sync(0xffffffffu, b, m ? __ffs(m) - 1 : 0);
    if (lane == 0) {
        int32_t out = TAU_OPEN;
        if (m) {
            // bin b >= 1 holds the scores v with (v - origin') * m31 >= b * 2^31, origin' = par.x / 2
            const int2 pr = par[q];
            const int64_t m31 = pr.y;
            const int64_t d_b = ((static_cast<int64_t>(bb) << 31) + m31 - 1) / m31;
            out = pr.x / 2 + static_cast<int32_t>(d_b);
        }
        tau[q] = out;
        if (theta0) theta0[q] = out;
    }
}

// Global candidate histogram (queue kernel): every key appended to ANY list of a query -- by any CTA -- bumps the
// bin of its score, measured from the query's seeded threshold.  Bins are only ever incremented for real,
// distinct documents, so "the bins >= b hold at least k candidates" proves that the k-th best score is at
// least theta0 + b * width: a threshold every list of the query may adopt, however few documents it has seen
// itself.  Lane l passes its 8 bins [8l, 8l + 8); returns b, or -1 while fewer than k candidates are known.
__device__ __forceinline__ int hist_bound(const uint4 &lo, const uint4 &hi, int k, int lane) {
    const uint32_t c[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t s = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) s += c[e];
    uint32_t suf = s;  // candidates in this lane's bins and all better ones
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += v;
    }
    const bool mine = suf >= static_cast<uint32_t>(k) && suf - s < static_cast<uint32_t>(k);
    int b = -1;
    if (mine) {
        uint32_t acc = suf - s;
#pragma unroll
        for (int e = 7; e >= 0; --e) {
            acc += c[e];
            if (b < 0 && acc >= static_cast<uint32_t>(k)) b = 8 * lane + e;
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, mine);
    return m ? __shfl_sync(0xffffffffu, b, __ffs(m) - 1) : -1;
}

// ================================================================================================
// Queue variant (main scans): the drain warps never maintain lists.  A score row whose maximum passes
// its query's threshold is parked in a shared-memory ring (8 STS.128 + a ticket) and two resolver warps
// turn parked rows into list entries, compact lists and publish tighter thresholds.  With only three
// accumulators in flight, any data-dependent pause of a drain warp used to stall the tensor pipe (the
// kernel above, still used for the open-threshold sample scans, ran at a third of its no-hit speed);
// here the accumulator hand-off takes the same time whatever the scores are.
// ================================================================================================
constexpr int Q_DRAIN = 12, Q_MMA_WARP = 12, Q_TMA_WARP = 13, Q_RES0 = 14, Q_RESOLVERS = 2;
constexpr int Q_THREADS = (Q_DRAIN + 2 + Q_RESOLVERS) * 32;  // 16 warps -> 128 registers per thread (four resolvers would cap it at 96: measured slower)
constexpr int RING_ROWS_MAX = 64;                             // parked rows per drain warp: Params::ring_rows = 32 or 64 (one vote can park 32)
constexpr int STASH_WORDS = 36;                               // a parked row: 32 scores, query, first document, ticket, pad (144 B)

struct QSmemLayout {
    uint32_t b_off, ring_off, state_off, hist_off, bar_off, total;
};
__host__ __device__ inline QSmemLayout q_smem_layout(int C, int NS, int ring_rows) {
    QSmemLayout L;
    uint32_t off = 0;
    L.b_off = off; off += static_cast<uint32_t>(NS) * STAGE_DOCS * 128 * C;
    L.ring_off = off; off += Q_DRAIN * ring_rows * STASH_WORDS * 4;
    L.state_off = off; off += 5 * 256 * 4 + 2 * Q_DRAIN * 4 + 32;  // per query: count, threshold, Dq, claim, seeded threshold; per drain warp: tail, final ticket
    L.hist_off = off; off += Q_RESOLVERS * 256 * 4;
    L.bar_off = off; off += (2 * NS + 2 * ACC_BUFS_MAX) * 8 + 16;
    L.total = off + 1024;
    return L;
}
// Ring hand-off words (tickets, consumption counters): release stores / acquire loads at CTA scope -- the PTX memory
// model's own ordering of the row payload against the word that publishes it (no volatile + fence pairs).  An mbarrier
// per ring slot (arrive.release / test_wait.acquire) was measured: same guarantees, but the resolvers' 32 barrier tests
// per ring and sweep cost 23 % of the 10k-query scan (14.55 -> 17.85 ms), and compute-sanitizer's racecheck flags the
// mbarrier form of this protocol as well (tools/sanitizer_probe.cu variant 5, profiles/README.md).
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

template <int C, int MT, bool DIRECT = false, int KP = 1>
__global__ void __launch_bounds__(Q_THREADS, 1) scan_queue_kernel(const Params p) {
    constexpr int B_STAGE = STAGE_DOCS * 128 * C;
    constexpr int KSTEPS = 4 * C;
    constexpr int EPI_PER_BUF = 8;                    // arrivals that free an accumulator: two column halves x four lane quarters
    constexpr int A_COLS = 32 * C * KP;               // tensor-memory columns of one 128-query operand tile (all K parts)
    constexpr int AB = KP == 1 ? ACC_BUFS_MAX : 2;    // accumulators: the operand of a two-part tile takes up to 256 columns
    constexpr int ACOL0 = AB * STAGE_DOCS;
    static_assert(KP == 1 || MT == 1, "two-part tiles leave room for one query tile");
    constexpr int NQ_CTA = 128 * MT;                  // queries of one group
    extern __shared__ unsigned char smem_unaligned[];
    const uint32_t pad = (1024u - (smem_u32(smem_unaligned) & 1023u)) & 1023u;
    unsigned char *smem = smem_unaligned + pad;
    const int NS = p.NS;
    const int RING_ROWS = p.ring_rows;
    const QSmemLayout L = q_smem_layout(C, NS, RING_ROWS);
    unsigned char *sB = smem + L.b_off;
    uint32_t *rings = reinterpret_cast<uint32_t *>(smem + L.ring_off);
    int *cnt_s = reinterpret_cast<int *>(smem + L.state_off), *theta_s = cnt_s + 256, *dq_s = cnt_s + 512, *claim_s = cnt_s + 768;
    int *theta0_s = cnt_s + 1024;
    int *tail_s = cnt_s + 1280, *fin_s = tail_s + Q_DRAIN;  // per drain warp: rows consumed by its resolver; final ticket of a segment
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bar_off);
    uint64_t *b_full = bars, *b_empty = bars + NS, *acc_full = bars + 2 * NS, *acc_empty = bars + 2 * NS + AB;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NS + 2 * AB);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    Items sg{static_cast<int64_t>(blockIdx.x), static_cast<int64_t>(p.n_seg) * p.groups, static_cast<int64_t>(gridDim.x),
             p.groups, p.seg_stages, static_cast<int>(p.stages), 0, 0, 0, 0};

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
        for (int i = 0; i < AB; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], EPI_PER_BUF); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int w = 0; w < Q_DRAIN; ++w) { tail_s[w] = 0; fin_s[w] = -1; }
    }
    for (int i = threadIdx.x; i < Q_DRAIN * RING_ROWS; i += Q_THREADS) rings[i * STASH_WORDS + 34] = 0u;  // no ticket yet
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    fence_before();
    cta_sync();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    uint32_t s_run = 0;
    const bool prof = p.prof != nullptr;
    long long w0 = 0, w1 = 0, w3 = 0, w5 = 0;
    int w2 = 0;
    const long long t_begin = prof ? clock64() : 0;
    uint64_t *group_lists = p.lists + static_cast<int64_t>(blockIdx.x) * NQ_CTA * static_cast<int64_t>(p.cap);
    // End of an item, after the resolvers have drained every ring: the 14 drain + resolver warps emit the
    // group's lists round-robin (<= k best keys each, unsorted, KEY_INF padded).  With two warps doing it, short
    // items (few query groups -> many document slices) spent more time emitting than scanning.
    auto emit_lists = [&](int slot, int *hist, int gr, int part) {
        const int64_t gq0 = static_cast<int64_t>(gr) * NQ_CTA;
        const int cap = p.cap, k = p.k;
        if constexpr (DIRECT) {  // one work item per CTA: leave the lists in place, publish their lengths
            for (int qc = slot * 32 + lane; qc < NQ_CTA; qc += (Q_DRAIN + Q_RESOLVERS) * 32)
                p.list_counts[static_cast<int64_t>(blockIdx.x) * NQ_CTA + qc] = gq0 + qc < p.nq ? cnt_s[qc] : 0;
            return;
        }
        for (int qc = slot; qc < NQ_CTA; qc += Q_DRAIN + Q_RESOLVERS) {
            const int64_t qq = gq0 + qc;
            if (qq >= p.nq) break;
            int c = cnt_s[qc];
            uint64_t *lrow = group_lists + static_cast<int64_t>(qc) * cap;
            if (c > k) { select_any(lrow, c, k, hist, lane); c = k; }
            __syncwarp();
            uint64_t *dst = p.out + (static_cast<int64_t>(part) * p.nq + qq) * k;
            for (int e = lane; e < k; e += 32) dst[e] = e < c ? __ldcg(lrow + e) : KEY_INF;
        }
        __syncwarp();
    };

    if (warp < Q_DRAIN) {
        // ================================ drain ================================
        // Drain warps keep no per-query state (thresholds live in shared memory, lists belong to the
        // resolvers), so accumulators are dealt to them round-robin: the four warps (one per TMEM lane
        // quarter) of set j serve accumulator buffer j, whichever query tile it holds.  Three sets give
        // every warp three MMA group times per accumulator.
        const int q4 = warp & 3, set = warp >> 2;
        uint32_t *ring = rings + warp * (RING_ROWS * STASH_WORDS);  // this warp's ring; resolver (q4 & 1) owns its queries' lists
        int head = 0, tail_seen = 0;                  // tickets handed out (warp-uniform) / consumption last observed
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
        while (sg.next()) {
            if (warp < 4 * MT) {  // query rows -> tensor memory; the queries' shared state
                const int mt = warp >> 2;
                const int qloc = mt * 128 + q4 * 32 + lane;
                const int64_t myq = static_cast<int64_t>(sg.gr) * NQ_CTA + qloc;
                const bool valid = myq < p.nq;
                const uint4 *src = reinterpret_cast<const uint4 *>(p.qimg + myq * (128 * C * KP));
                const uint32_t ta = lane_base + ACOL0 + mt * A_COLS;
#pragma unroll
                for (int c = 0; c < A_COLS / 8; ++c) tmem_st8(ta + c * 8, __ldg(src + 2 * c), __ldg(src + 2 * c + 1));
                tmem_st_wait();
                cnt_s[qloc] = 0;
                dq_s[qloc] = valid ? p.qconst[myq] : 0;
                theta_s[qloc] = valid ? (p.tau_init ? max(TAU_OPEN, p.tau_init[myq]) : TAU_OPEN) : TAU_NEVER;
                theta0_s[qloc] = (valid && p.theta0) ? max(TAU_OPEN, p.theta0[myq]) : TAU_OPEN;
            }
            fence_before();
            cta_sync();

            // 32 scores of one query row: 3-input max tree, one compare, one vote; a row whose maximum passes is
            // parked for the resolver (its scores, its query, its first document, a ticket)
            auto max32 = [](const int (&v)[32]) { return max(max(max8(v), max8(v + 8)), max(max8(v + 16), max8(v + 24))); };
            auto filter = [&](const int (&v)[32], int m, int theta, int qloc, uint32_t doc0) {   // m = max32(v)
                const bool hit = m >= theta;
                const unsigned hm = __ballot_sync(0xffffffffu, hit);
                if (hm) {
                    ++w1;
                    const long long th0 = prof ? clock64() : 0;
                    const int n = __popc(hm);
                    const int t0 = head;
                    head += n;
                    if (head - tail_seen > RING_ROWS) {  // maybe full: look at the resolver's progress, wait if it is behind
                        const long long tw = prof ? clock64() : 0;
#ifdef XFBQ_UMMA_WATCHDOG
                        const long long wd0 = clock64();
#endif
                        while (head - (tail_seen = ld_acquire(&tail_s[warp])) > RING_ROWS) {
                            __nanosleep(40);
#ifdef XFBQ_UMMA_WATCHDOG
                            if (clock64() - wd0 > 4000000000ll) { if (lane == 0) printf("drain %d cta %d stuck: head %d tail %d\n", warp, blockIdx.x, head, tail_seen); __trap(); }
#endif
                        }
                        if (prof) w3 += clock64() - tw;
                    }
                    if (p.debug & 64) { head = t0; }  // timing experiments: evaluate the filter, park nothing
                    else if (hit) {
                        const int t = t0 + __popc(hm & ((1u << lane) - 1u));
                        uint32_t *row = ring + (t & (RING_ROWS - 1)) * STASH_WORDS;
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            *reinterpret_cast<uint4 *>(row + 4 * c) = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                        row[32] = qloc;
                        row[33] = doc0;
                        if (p.debug & 16) *reinterpret_cast<volatile int *>(row + 34) = t + 1;  // timing experiments: no release fence
                        else st_release(reinterpret_cast<int *>(row + 34), t + 1);  // publishes the row
                    }
                    __syncwarp();
                    if (prof) w5 += clock64() - th0;
                }
            };

            const uint32_t u_begin = s_run * MT, u_end = u_begin + static_cast<uint32_t>(sg.cnt) * MT;
            {
                // Half accumulators dealt round-robin to the three warps of a lane quarter: 64 columns are in registers after
                // one tensor-memory read, so the buffer goes back to the issuer BEFORE any filtering -- parking a row never
                // delays the tensor pipe, and the hand-off chain is one read round instead of two reads and two filters.
                const uint32_t n_units = 2 * (u_end - u_begin);
                for (uint32_t x = set; x < n_units; x += 3) {
                    const uint32_t rel = x >> 1, half = x & 1u;
                    const uint32_t u = u_begin + rel;
                    const uint32_t buf = u % AB;
                    const int mt = MT == 2 ? static_cast<int>(rel & 1u) : 0;
                    const int qloc = mt * 128 + q4 * 32 + lane;
                    const uint32_t doc0 = (static_cast<uint32_t>(sg.sd0) + rel / MT) * STAGE_DOCS + half * 64;
                    const uint32_t taddr = lane_base + buf * STAGE_DOCS + half * 64;
                    const int theta = theta_s[qloc];
                    asm volatile("" ::"r"(taddr), "r"(doc0), "r"(theta));   // computed BEFORE the wait: between the barrier and the tensor-memory read only the read itself
                    if (prof) mbar_wait_prof(&acc_full[buf], (u / AB) & 1u, true, w0); else mbar_wait_tight(&acc_full[buf], (u / AB) & 1u);
                    fence_after();
                    int v[2][32];
                    tmem_ld32(taddr, v[0]);
                    tmem_ld32(taddr + 32, v[1]);
                    tmem_ld_wait();
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&acc_empty[buf]);
                    if (!(p.debug & 4)) {   // one vote for the 64 columns: the common case (nothing passes) costs two max trees, a compare and a vote
                        const int m0 = max32(v[0]), m1 = max32(v[1]);
                        if (__any_sync(0xffffffffu, max(m0, m1) >= theta)) {
                            filter(v[0], m0, theta, qloc, doc0);
                            filter(v[1], m1, theta, qloc, doc0 + 32);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) st_release(&fin_s[warp], head);  // every ticket of this segment is out
            cta_sync();  // the resolvers have emptied the rings: lists are final, this warp's ring is free scratch
            emit_lists(warp, reinterpret_cast<int *>(ring), sg.gr, sg.part);
            __syncwarp();
            for (int i = lane; i < RING_ROWS; i += 32) ring[i * STASH_WORDS + 34] = 0u;  // scratch use may have forged tickets
            head = 0; tail_seen = 0;
            if (lane == 0) { st_release(&tail_s[warp], 0); }
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
        if (prof && threadIdx.x == 0) {
            unsigned long long *o = p.prof + blockIdx.x * 8;
            o[0] = w0; o[1] = w1; o[5] = w3; o[6] = clock64() - t_begin; o[7] = s_run;
        }
        if (prof && lane == 0) {   // every drain warp's time waiting for an accumulator / for room in its ring
            p.prof[gridDim.x * 12 + blockIdx.x * 12 + warp] = w0;
            p.prof[gridDim.x * 24 + blockIdx.x * 12 + warp] = w3;
            p.prof[gridDim.x * 36 + blockIdx.x * 24 + warp] = w5;        // time inside the park path ...
            p.prof[gridDim.x * 36 + blockIdx.x * 24 + 12 + warp] = w1;   // ... of this many chunks
        }
    } else if (warp == Q_MMA_WARP) {
        // ================================ MMA issuer ================================
        const uint32_t b_lo0 = desc_lo(smem_u32(sB));
        if (tmem != 0u) __trap();  // the CTA owns all 512 columns: the allocation starts at lane 0, column 0 (addresses below rely on it)
        constexpr uint32_t tm = 0u;
        while (sg.next()) {
            cta_sync();
            fence_after();
            Ring rb{static_cast<int>((s_run * KP) % NS), ((s_run * KP) / NS) & 1u};
            const uint32_t u0 = s_run * MT;
            Ring ac{static_cast<int>(u0 % AB), ((u0 / AB) & 1u) ^ 1u};
            if constexpr (KP > 1) {
            for (int i = 0; i < sg.cnt; ++i) {
                if constexpr (KP > 1) {  // one accumulator per tile, fed by KP operand stages
                    const uint32_t buf = ac.idx;
                    mbar_wait_prof(&acc_empty[buf], ac.phase, prof, w1);
                    fence_after();
#pragma unroll
                    for (int part = 0; part < KP; ++part) {
                        if (prof) mbar_wait_prof(&b_full[rb.idx], rb.phase, true, w0); else mbar_wait_tight(&b_full[rb.idx], rb.phase);
                        fence_after();
                        const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(rb.idx) * (B_STAGE >> 4);
                        if (elect_one()) {
                            const uint32_t d = tm + buf * STAGE_DOCS;
#pragma unroll
                            for (int ks = 0; ks < KSTEPS; ++ks) {
                                const uint32_t ta = tm + ACOL0 + (part * KSTEPS + ks) * 8;
                                const uint32_t bo = ((ks >> 2) * (STAGE_DOCS * 128) + (ks & 3) * 32) >> 4;
                                if (part == 0 && ks == 0) umma_i8<false>(d, ta, b_lo + bo);
                                else umma_i8<true>(d, ta, b_lo + bo);
                            }
                            umma_commit(&b_empty[rb.idx]);
                            if (part == KP - 1) umma_commit(&acc_full[buf]);
                        }
                        __syncwarp();
                        rb.advance(NS);
                    }
                    ac.advance(AB);
                }
            }
            } else {
            // One tile = MT groups of KSTEPS MMAs.  Whatever the issuing warp executes between the last tcgen05.mma of a group
            // and the first of the next is NOT hidden behind the MMAs it has queued (tools/umma_probe.cu tests 10-12: in a steady
            // stream the tensor pipe accepts an MMA only about when it can start it, so a dependent chain between two groups adds
            // its full length to every group), but what sits between two MMAs of the SAME group is free as long as it fits one
            // MMA time (64 clk).  So the barrier waits of the NEXT group are placed in the middle of the current one, the second half
            // of a group and the first half of the next are issued from one elected block, and every operand of the MMAs is computed from warp-uniform values only
            // (tensor memory starts at column 0: checked after the allocation), which keeps them in uniform registers -- the
            // R2UR moves of the first version were the longest part of the gap.
            auto wait_operand = [&](const Ring &r) { if (prof) mbar_wait_prof(&b_full[r.idx], r.phase, true, w0); else mbar_wait_tight(&b_full[r.idx], r.phase); };
            auto wait_acc = [&](const Ring &r) { if (prof) mbar_wait_prof(&acc_empty[r.idx], r.phase, true, w1); else mbar_wait_tight(&acc_empty[r.idx], r.phase); };
            auto mmas = [&](uint32_t d, uint32_t ta0, uint32_t b_lo, int ks0, int ks1) {
#pragma unroll
                for (int ks = 0; ks < KSTEPS; ++ks)
                    if (ks >= ks0 && ks < ks1) {
                        const uint32_t bo = ((ks >> 2) * (STAGE_DOCS * 128) + (ks & 3) * 32) >> 4;
                        if (ks == 0) umma_i8<false>(d, ta0 + ks * 8, b_lo + bo);
                        else umma_i8<true>(d, ta0 + ks * 8, b_lo + bo);
                    }
            };
            constexpr int H = KSTEPS - 1;   // MMAs of a group issued from the earlier block: the later the probe for the next group's
                                            // accumulator, the more time its drain has had (H = 4 / 6 / 7 of 8: 1 152 / 1 143 / 1 120 clk per tile)
            // Rotated loop: an elected block issues the last MMA of one group, its commit(s) and the first MMAs of the NEXT
            // group back to back, so every group boundary lies inside a block; the gaps between blocks (barrier polls, elect,
            // uniform-register set-up) fall between two MMAs of the same group.  The next group's barriers are only PROBED in
            // the middle of a group: when its accumulator or operand tile is not there yet (short rings, the HBM-bound batch
            // sizes) the current group is finished and committed first -- holding its second half back would delay the
            // release of its own operand stage -- and the next group starts from its own block after a blocking wait.
            auto ready = [&](uint64_t *bar, uint32_t parity) {   // warp-uniform: every lane reads the same barrier
                uint32_t ok;
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
                return __all_sync(0xffffffffu, ok != 0);
            };
            if (sg.cnt > 0) {
                wait_operand(rb); wait_acc(ac); fence_after();
                if (elect_one()) mmas(static_cast<uint32_t>(ac.idx) * STAGE_DOCS, ACOL0, b_lo0 + static_cast<uint32_t>(rb.idx) * (B_STAGE >> 4), 0, H);
                __syncwarp();
            }
            for (int i = 0; i < sg.cnt; ++i) {
                uint32_t tz;   // a zero neither compiler can see through or hoist: tensor-memory addresses below are `tz + constant`, so ptxas moves ONE
                               // register to the uniform datapath per block and adds the constants there instead of eight R2UR
                asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(tz) : "r"(smem_u32(tmem_slot)));  // the allocation's base: 0 (checked above)
                const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(rb.idx) * (B_STAGE >> 4);
                const uint32_t d0 = static_cast<uint32_t>(ac.idx) * STAGE_DOCS;
                uint64_t *stage_done = &b_empty[rb.idx];
                uint64_t *acc0_done = &acc_full[ac.idx];
                const bool more = i + 1 < sg.cnt;
                ac.advance(AB);
                rb.advance(NS);
                uint32_t d1 = 0;
                uint64_t *acc1_done = nullptr;
                if constexpr (MT == 2) {
                    d1 = static_cast<uint32_t>(ac.idx) * STAGE_DOCS;
                    acc1_done = &acc_full[ac.idx];
                    if (ready(&acc_empty[ac.idx], ac.phase)) {   // the second query tile's accumulator is free: one block
                        fence_after();
                        if (elect_one()) {
                            mmas(d0, tz + ACOL0, b_lo, H, KSTEPS);
                            umma_commit(acc0_done);
                            mmas(d1, tz + ACOL0 + A_COLS, b_lo, 0, H);
                        }
                        __syncwarp();
                    } else {
                        ++w2;   // profiling: the second query tile's accumulator was not free at the probe
                        if (elect_one()) { mmas(d0, tz + ACOL0, b_lo, H, KSTEPS); umma_commit(acc0_done); }
                        __syncwarp();
                        wait_acc(ac);
                        fence_after();
                        if (elect_one()) mmas(d1, tz + ACOL0 + A_COLS, b_lo, 0, H);
                        __syncwarp();
                    }
                    ac.advance(AB);
                }
                // second half of the tile's last group, the commits, and -- when it can start -- the first half of the next tile
                const uint32_t dl = MT == 2 ? d1 : d0;
                const uint32_t al = tz + (MT == 2 ? ACOL0 + A_COLS : ACOL0);
                uint64_t *accl_done = MT == 2 ? acc1_done : acc0_done;
                const uint32_t dn = static_cast<uint32_t>(ac.idx) * STAGE_DOCS;
                const uint32_t bn = b_lo0 + static_cast<uint32_t>(rb.idx) * (B_STAGE >> 4);
                if (more && ready(&b_full[rb.idx], rb.phase) && ready(&acc_empty[ac.idx], ac.phase)) {
                    fence_after();
                    if (elect_one()) {
                        mmas(dl, al, b_lo, H, KSTEPS);
                        umma_commit(accl_done);
                        umma_commit(stage_done);
                        mmas(dn, tz + ACOL0, bn, 0, H);
                    }
                    __syncwarp();
                } else {
                    if (more) w2 += 1 << 16;   // profiling: the next tile's operand or accumulator was not there at the probe
                    if (elect_one()) { mmas(dl, al, b_lo, H, KSTEPS); umma_commit(accl_done); umma_commit(stage_done); }
                    __syncwarp();
                    if (more) {
                        wait_operand(rb); wait_acc(ac); fence_after();
                        if (elect_one()) mmas(dn, tz + ACOL0, bn, 0, H);
                        __syncwarp();
                    }
                }
            }
            }
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();  // lists final
            cta_sync();  // lists emitted
        }
        if (prof && lane == 0) {
            p.prof[blockIdx.x * 8 + 2] = w0; p.prof[blockIdx.x * 8 + 3] = w1;
            p.prof[gridDim.x * 8 + blockIdx.x * 4 + 0] = static_cast<unsigned>(w2) & 0xFFFFu;   // probes that failed: second query tile ...
            p.prof[gridDim.x * 8 + blockIdx.x * 4 + 1] = static_cast<unsigned>(w2) >> 16;        // ... next document tile
        }
    } else if (warp == Q_TMA_WARP) {
        // ================================ loader ================================
        const unsigned char *db = reinterpret_cast<const unsigned char *>(p.db);
        while (sg.next()) {
            cta_sync();
            if (lane == 0) {
                Ring rb{static_cast<int>((s_run * KP) % NS), (((s_run * KP) / NS) & 1u) ^ 1u};
                for (int i = 0; i < sg.cnt; ++i) {
#pragma unroll
                    for (int part = 0; part < KP; ++part) {
                        mbar_wait_prof(&b_empty[rb.idx], rb.phase, prof, w0);
                        mma::mbar_arrive_expect_tx(&b_full[rb.idx], B_STAGE);
                        mma::tma_bulk_g2s(sB + static_cast<size_t>(rb.idx) * B_STAGE,
                                          db + (static_cast<int64_t>(sg.sd0 + i) * KP + part) * B_STAGE, B_STAGE, &b_full[rb.idx]);
                        rb.advance(NS);
                    }
                }
            }
            __syncwarp();
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();  // lists final
            cta_sync();  // lists emitted
        }
        if (prof && lane == 0) { p.prof[blockIdx.x * 8 + 4] = w0; }
    } else {
        // ================================ resolvers ================================
        const int res = warp - Q_RES0;
        int *hist = reinterpret_cast<int *>(smem + L.hist_off) + res * 256;
        const uint32_t n_docs = static_cast<uint32_t>(p.n);
        const uint32_t id_off = static_cast<uint32_t>(p.row_offset);
        const int cap = p.cap, k = p.k;
        while (sg.next()) {
            cta_sync();
            const int64_t gq0 = static_cast<int64_t>(sg.gr) * NQ_CTA;
            int idle = 0;
            // round-robin refresh of this resolver's queries from the global histogram: the bins of the next query
            // are fetched while the current sweep runs (one L2 round trip per sweep would double its length)
            constexpr int OWN_Q = NQ_CTA / Q_RESOLVERS;
            // The CTAs that scan this query group at the same time (one per document slice) start their rounds at different
            // queries, so between them every query's histogram is read every few sweeps; what one CTA proves it publishes
            // through theta_g, and every CTA imports theta_g for all its queries every few sweeps (below).  A lone CTA
            // gets round to a query only every OWN_Q sweeps: with one query group (<= 256 queries, 148 slices of 0.6 ms)
            // thresholds lagged so far behind that 31 % of the 32 x 32 score chunks parked a row.
            int rq = static_cast<int>((static_cast<int64_t>(sg.part) * OWN_Q) / (p.n_seg > 0 ? p.n_seg : 1)) % OWN_Q, rq_pending = -1;
            int sweeps = 0;
            uint4 hb_lo = make_uint4(0u, 0u, 0u, 0u), hb_hi = hb_lo;
#ifdef XFBQ_UMMA_WATCHDOG
            long long wd0 = clock64();
#endif
            while (true) {
                if (p.ghist) {
                    if (rq_pending >= 0) {
                        const int b = hist_bound(hb_lo, hb_hi, k, lane);
                        if (b > 0 && lane == 0) {
                            const int th = theta0_s[rq_pending] + (b << p.hist_shift);
                            if (th > theta_s[rq_pending]) {
                                atomicMax(&theta_s[rq_pending], th);
                                if (p.theta_g) atomicMax(p.theta_g + gq0 + rq_pending, th);
                            }
                        }
                    }
                    const int qn = (res + Q_RESOLVERS * (rq >> 5)) * 32 + (rq & 31);  // the queries of this resolver's blocks in turn
                    rq = rq + 1 == OWN_Q ? 0 : rq + 1;
                    if (gq0 + qn < p.nq) {
                        const uint4 *bins = reinterpret_cast<const uint4 *>(p.ghist + (gq0 + qn) * HIST_BINS) + 2 * lane;
                        hb_lo = __ldcg(bins);
                        hb_hi = __ldcg(bins + 1);
                        rq_pending = qn;
                    } else {
                        rq_pending = -1;
                    }
                }
                bool progressed = false;
                bool all_done = true;
#pragma unroll 1
                for (int w = res; w < Q_DRAIN; w += Q_RESOLVERS) {  // the rings of the drain warps this resolver serves
                    uint32_t *ring = rings + w * (RING_ROWS * STASH_WORDS);
                    const int tail = ld_acquire(&tail_s[w]);
                    // rows tail .. tail + n - 1 are ready (tickets are handed out in order, rows may land out of order)
                    const int t = tail + lane;
                    const uint32_t *row = ring + (t & (RING_ROWS - 1)) * STASH_WORDS;
                    const bool ready = ld_acquire(reinterpret_cast<const int *>(row + 34)) == t + 1;
                    const unsigned rm = __ballot_sync(0xffffffffu, ready);
                    const int n = rm == 0xffffffffu ? 32 : __ffs(~rm) - 1;
                    if (n == 0) {
                        if (ld_acquire(&fin_s[w]) != tail) all_done = false;
                        continue;
                    }
                    progressed = true;
                    all_done = false;
                    bool pend = lane < n;
                    const int q = pend ? static_cast<int>(row[32]) : 0;
                    const uint32_t doc0 = pend ? row[33] : 0u;
                    while (__any_sync(0xffffffffu, pend)) {
                        // a round adds at most 32 keys to a list:
// one row per query and round: the last lane to claim the query's word goes (an atomic exchange, so the lanes' writes
                        // are ordered; __match_any_sync picks the same kind of winner but cost 2 % of the 10k-query scan)
                        if (pend) atomicExch(&claim_s[q], lane);
                        __syncwarp();
                        const bool go = pend && claim_s[q] == lane;
                        if (go && (p.debug & 8)) pend = false;  // timing experiments: parked rows are dropped unread
                        else if (go) {
                            const int th = theta_s[q], dqe = dq_s[q];
                            uint32_t below = 0;  // bit j: score j < threshold
#pragma unroll
                            for (int c = 7; c >= 0; --c) {
                                const uint4 sw = *reinterpret_cast<const uint4 *>(row + 4 * c);
                                below = __funnelshift_l(sw.w - static_cast<uint32_t>(th), below, 1);
                                below = __funnelshift_l(sw.z - static_cast<uint32_t>(th), below, 1);
                                below = __funnelshift_l(sw.y - static_cast<uint32_t>(th), below, 1);
                                below = __funnelshift_l(sw.x - static_cast<uint32_t>(th), below, 1);
                            }
                            uint32_t hits = ~below;
                            uint64_t *list = group_lists + static_cast<int64_t>(q) * cap;
                            int c = cnt_s[q];
                            while (hits) {
                                const int j = __ffs(hits) - 1;
                                hits &= hits - 1;
                                const uint32_t doc = doc0 + j;
                                if (doc < n_docs) {
                                    const int val = static_cast<int>(row[j]);
                                    list[c++] = (static_cast<uint64_t>(static_cast<uint32_t>(dqe - val)) << 32) | (id_off + doc);
                                    if (p.ghist) atomicAdd(p.ghist + (gq0 + q) * HIST_BINS + min((val - theta0_s[q]) >> p.hist_shift, HIST_BINS - 1), 1u);
                                }
                            }
                            cnt_s[q] = c;
                            pend = false;
                        }
                        __syncwarp();
                        unsigned need = __ballot_sync(0xffffffffu, go && cnt_s[q] > cap - 32);
                        while (need) {  // a list that another row could overflow: keep its k best, tighten its threshold
                            const int src = __ffs(need) - 1;
                            need &= need - 1;
                            const int qc = __shfl_sync(0xffffffffu, q, src);
                            ++w2;
                            const uint64_t kth = select_any(group_lists + static_cast<int64_t>(qc) * cap, cnt_s[qc], k, hist, lane);
                            if (lane == src) {
                                cnt_s[qc] = k;
                                const int th = dq_s[qc] - static_cast<int>(kth >> 32);
                                atomicMax(&theta_s[qc], th);
                                if (p.theta_g && gq0 + qc < p.nq) atomicMax(p.theta_g + gq0 + qc, th);  // every CTA scanning this query tightens with us
                            }
                            __syncwarp();
                        }
                    }
                    __syncwarp();
                    if (lane == 0) st_release(&tail_s[w], tail + n);
                    __syncwarp();
                }
                if (all_done) break;
#ifdef XFBQ_UMMA_WATCHDOG
                if (progressed) wd0 = clock64();
                else if (clock64() - wd0 > 4000000000ll) {
                    if (lane == 0) {
                        printf("resolver %d cta %d stuck:", res, blockIdx.x);
                        for (int w = res; w < Q_DRAIN; w += Q_RESOLVERS) printf(" [w%d tail %d fin %d flag %d addr %u]", w, tail_s[w], fin_s[w], (int)rings[(w * RING_ROWS + (tail_s[w] & (RING_ROWS - 1))) * STASH_WORDS + 34], smem_u32(&rings[(w * RING_ROWS + (tail_s[w] & (RING_ROWS - 1))) * STASH_WORDS + 34]));
                        printf("\n");
                    }
                    __trap();
                }
#endif
                if (p.theta_g && ((++sweeps & 7) == 0 || (!progressed && (++idle & 15) == 0))) {
                    // import the thresholds other CTAs found for our queries (4 coalesced loads per resolver)
                    for (int blk = res; blk < NQ_CTA / 32; blk += Q_RESOLVERS) {
                        const int qc = blk * 32 + lane;
                        if (gq0 + qc < p.nq) {
                            const int th = __ldcg(p.theta_g + gq0 + qc);
                            if (th > theta_s[qc]) atomicMax(&theta_s[qc], th);
                        }
                    }
                }
                if (!progressed) __nanosleep(100);
            }
            cta_sync();  // every resolver is done: lists are final
            emit_lists(Q_DRAIN + res, hist, sg.gr, sg.part);
            if (lane < Q_DRAIN && (lane % Q_RESOLVERS) == res) st_release(&fin_s[lane], -1);  // next segment's tickets are not out yet
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
        if (prof && lane == 0 && res == 0) { p.prof[gridDim.x * 8 + blockIdx.x * 4 + 2] = w2; }
    }
    fence_before();
    cta_sync();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace umma
