// xfbq_umma.cuh -- tcgen05 (5th-generation tensor core) scan engine (included by xfbq_b200.cu).
//
// Same arithmetic as the IMMA engine (xfbq_mma.cuh): the XOR/popcount distance of _kernels.py:56-69
// is the exact integer form  d = Dq - sum_k x_k (2 y_k - Aq);  here the s8 x s8 -> s32 dot products
// run on tcgen05.mma.kind::i8 (measured 8 188 MAC/clk/SM, 4x the mma.sync IMMA pipe) with the
// accumulators in tensor memory.
//
// One persistent CTA per SM, 16 warps (13 working) in three roles that only meet at mbarriers:
//   producers (4 warps)  nibble layout (row-major 4-bit codes, 64C bytes per document) -> registers
//                        (two stages of LDG.128 in flight) -> split nibbles to bytes -> the B operand
//                        stage in shared memory: 128 documents x 128C bytes, K-major, 128-byte swizzle
//                        (the canonical UMMA layout, written with conflict-free STS.128)
//   issuer (1 thread)    per stage and per 128-query tile: 4C x tcgen05.mma (M = 128 queries, N = 128
//                        documents, K = 32) into one of four 128-column TMEM accumulators;
//                        tcgen05.commit releases the operand stage / publishes the accumulator
//   epilogue (8 warps)   tcgen05.ld 32 lanes x 32 columns: a thread owns ONE query row, so its threshold
//                        is a register and its candidate list is private: 3-input max over the 32
//                        scores, compare once, and only on a hit append (distance << 32 | row id) keys;
//                        a list that could overflow is cut to its k best by a warp-level radix select
//                        (search.py:129-131 order on the full key), which also tightens the threshold.
// The query operand (s8 weights 2y - Aq in the same K permutation the producers emit) is staged once
// per query group as a ready-made swizzled image (prep_queries_kernel).  Work = groups x stages is
// linearised and cut into gridDim.x equal ranges, as in the IMMA engine.
#pragma once

namespace umma {

constexpr int EPI_WARPS = 8;    // warpgroups 0-1
constexpr int PROD_WARPS = 4;   // warpgroup 2
constexpr int MMA_WARP = 12;    // first warp of warpgroup 3 (its other three warps only take part in block barriers)
constexpr int THREADS = 512;    // whole warpgroups, so that setmaxnreg can move registers between the roles
constexpr int EPI_REGS = 168, PROD_REGS = 104, MMA_REGS = 40;  // 8*168 + 4*104 + 4*40 = 1920 <= 2048 per lane slot
constexpr int STAGE_DOCS = 128;  // N of one MMA
constexpr int ACC_BUFS = 4;      // 4 x 128 columns = the whole tensor memory
constexpr int TAU_OPEN = -(1 << 30);
constexpr int TAU_NEVER = 1 << 30;     // |acc| <= 512 * 15 * 127 < 2^20, so acc - tau never overflows

struct Params {
    const void *db;            // nibble layout
    int64_t n, n_pad, row_offset;
    const unsigned char *qimg; // [groups][MT][C][128 rows x 128 B, swizzled] s8 weights
    const int32_t *qconst;     // [nq_pad] Dq
    const int32_t *tau_init;   // [nq] or nullptr
    uint64_t *lists;           // [grid][EPI_WARPS][32][cap]
    uint64_t *out;             // [slots * DW][nq][k], KEY_INF pre-filled when slots > 1
    int64_t nq, stages;
    int groups, k, cap, NS;    // NS = operand stages in shared memory
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
// Shared-memory operand descriptor, K-major, SWIZZLE_128B: rows of 128 bytes, 8-row groups 1024 B apart
// (start address >> 4 | LBO (unused) | SBO = 1024 >> 4 | version 1 | layout type 2).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor: D = s32, A = B = signed 8-bit, both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(STAGE_DOCS >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate) : "memory");
}
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
template <int R> __device__ __forceinline__ void reg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R)); }
template <int R> __device__ __forceinline__ void reg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R)); }

__device__ __forceinline__ int tmem_ld1(uint32_t taddr) {
    int v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
    return v;
}
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 0;" ::: "memory"); }
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
// dim = 32g + e + 4hi + 8j.  The image is exactly what the MMA reads from shared memory.
__global__ void __launch_bounds__(256)
prep_queries_kernel(const uint32_t *__restrict__ q, int64_t nq, int64_t nq_pad, int dim, int wq, int wd, int C, int MT,
                    unsigned char *__restrict__ qimg, int32_t *__restrict__ qconst) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= nq_pad) return;
    const int W = 4 * C;
    const int Aq = (1 << wq) - 1, Ad = (1 << wd) - 1;
    const int64_t tile = row >> 7;  // = group * MT + mt
    const int r = static_cast<int>(row & 127);
    unsigned char *img = qimg + tile * (static_cast<int64_t>(C) * 128 * 128);
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
                int y = 0;
                for (int jq = 0; jq < wq; ++jq) y |= static_cast<int>((q[(row * wq + jq) * W + word] >> bit) & 1u) << jq;
                int w = 0;
                if (d < dim) { w = 2 * y - Aq; sy += y; }
                packed |= (static_cast<uint32_t>(w) & 0xFFu) << (8 * j);
            }
        }
        *reinterpret_cast<uint32_t *>(img + sw128_offset(r, 4 * ow, 128)) = packed;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sy += __shfl_xor_sync(0xffffffffu, sy, o);
    if (lane == 0) qconst[row] = (row < nq) ? Ad * sy : 0;
}

struct SmemLayout {
    uint32_t a_off, b_off, hist_off, bar_off, total;
};
__host__ __device__ inline SmemLayout smem_layout(int C, int MT, int NS) {
    SmemLayout L;
    uint32_t off = 0;
    L.a_off = off; off += static_cast<uint32_t>(MT) * 128 * 128 * C;
    L.b_off = off; off += static_cast<uint32_t>(NS) * STAGE_DOCS * 128 * C;
    L.hist_off = off; off += EPI_WARPS * 256 * 4;
    L.bar_off = off; off += (2 * NS + 2 * ACC_BUFS) * 8 + 16;
    L.total = off + 1024;  // slack for the manual 1024-byte alignment of the operand area
    return L;
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

template <int C, int MT>
__global__ void __launch_bounds__(THREADS, 1) scan_kernel(const Params p) {
    constexpr int ROW_BYTES = 64 * C;                 // one document in the nibble layout
    constexpr int A_TILE = 128 * 128 * C;             // one 128-query operand tile
    constexpr int B_STAGE = STAGE_DOCS * 128 * C;     // one document stage, bytes
    constexpr int KSTEPS = 4 * C;                     // K = 32 per MMA
    constexpr int DPI = 8 / C;                        // documents per producer warp-iteration (32 x 16 B)
    constexpr int ITW = (STAGE_DOCS / DPI) / PROD_WARPS;  // warp-iterations per producer warp per stage
    constexpr int COLS = MT == 2 ? 128 : 64;          // accumulator columns an epilogue warp drains
    constexpr int EPI_PER_BUF = MT == 2 ? 4 : 8;      // epilogue warps reading one accumulator
    extern __shared__ unsigned char smem_unaligned[];
    const uint32_t pad = (1024u - (smem_u32(smem_unaligned) & 1023u)) & 1023u;
    unsigned char *smem = smem_unaligned + pad;
    const int NS = p.NS;
    const SmemLayout L = smem_layout(C, MT, NS);
    unsigned char *sA = smem + L.a_off, *sB = smem + L.b_off;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bar_off);
    uint64_t *b_full = bars, *b_empty = bars + NS, *acc_full = bars + 2 * NS, *acc_empty = bars + 2 * NS + ACC_BUFS;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NS + 2 * ACC_BUFS);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const int64_t T = p.stages;
    const int64_t W = static_cast<int64_t>(p.groups) * T;
    const int64_t G = gridDim.x;
    Segments sg{static_cast<int64_t>(blockIdx.x) * W / G, (static_cast<int64_t>(blockIdx.x) + 1) * W / G, T, 0, 0, 0};

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&b_full[i], PROD_WARPS); mbar_init(&b_empty[i], 1); }
        for (int i = 0; i < ACC_BUFS; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], EPI_PER_BUF); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    fence_before();
    cta_sync();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // Every role runs the same segment loop:  stage the group's query operand (all threads, generic
    // proxy + proxy fence) | barrier | role work | barrier (every MMA that read the operand is done:
    // the epilogue has consumed its result).
    auto stage_queries = [&](int gr) {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.qimg + static_cast<int64_t>(gr) * MT * A_TILE);
        uint4 *dst = reinterpret_cast<uint4 *>(sA);
        for (int i = threadIdx.x; i < MT * A_TILE / 16; i += THREADS) dst[i] = __ldg(src + i);
        fence_async_smem();
    };
    uint32_t s_run = 0;  // stages this CTA has processed so far (drives every ring cursor)

    if (warp < EPI_WARPS) {
        // ================================ epilogue ================================
        reg_inc<EPI_REGS>();
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
            stage_queries(sg.gr);
            cta_sync();
            const int64_t q0 = (static_cast<int64_t>(sg.gr) * MT + mt) * 128 + q4 * 32;  // first query row of this warp
            const int64_t myq = q0 + lane;
            const bool valid = myq < p.nq;
            const int dq = valid ? p.qconst[myq] : 0;
            int theta = valid ? (p.tau_init ? max(TAU_OPEN, p.tau_init[myq]) : TAU_OPEN) : TAU_NEVER;
            int cnt = 0;

            // 32 scores of this thread's query row: 3-input max tree, one compare, one vote.  On a hit
            // (rare once thresholds have tightened) the warp builds per-lane hit masks from sign bits
            // and re-reads just the hit columns from tensor memory, so no score is indexed dynamically.
            auto filter = [&](const int (&v)[32], uint32_t taddr_c, uint32_t doc0) {
                const int g0 = max8(v), g1 = max8(v + 8), g2 = max8(v + 16), g3 = max8(v + 24);
                const int m = max(max(g0, g1), max(g2, g3));
                if (__any_sync(0xffffffffu, m >= theta)) {
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
                    uint32_t cols = __reduce_or_sync(0xffffffffu, hits);
                    while (cols) {
                        const int j = __ffs(cols) - 1;
                        cols &= cols - 1;
                        const int val = tmem_ld1(taddr_c + j);
                        tmem_ld_wait();
                        if (((hits >> j) & 1u) && doc0 + j < n_docs) {
                            my_list[cnt] = (static_cast<uint64_t>(static_cast<uint32_t>(dq - val)) << 32) | (id_off + doc0 + j);
                            ++cnt;
                        }
                    }
                    __syncwarp();
                    unsigned need = __ballot_sync(0xffffffffu, cnt > cap - 32);
                    while (need) {  // a list that the next 32 documents could overflow: keep its k best
                        const int ql = __ffs(need) - 1;
                        need &= need - 1;
                        const int c = __shfl_sync(0xffffffffu, cnt, ql);
                        const uint64_t kth = mma::select_row(warp_lists + static_cast<int64_t>(ql) * cap, c, k, hist, lane);
                        if (lane == ql) { cnt = k; theta = dq - static_cast<int>(kth >> 32); }
                    }
                }
            };

            for (int i = 0; i < sg.cnt; ++i) {
                const uint32_t u = (s_run + i) * MT + mt;
                const uint32_t buf = u & (ACC_BUFS - 1), use = u / ACC_BUFS;
                mbar_wait(&acc_full[buf], use & 1u);
                fence_after();
                const uint32_t taddr = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + buf * STAGE_DOCS + col0;
                const uint32_t doc0 = static_cast<uint32_t>(sg.sd0 + i) * STAGE_DOCS + col0;
                int va[32], vb[32];
                tmem_ld32(taddr, va);
                tmem_ld_wait();
#pragma unroll 1
                for (int c = 0; c < COLS / 32; c += 2) {
                    tmem_ld32(taddr + (c + 1) * 32, vb);
                    filter(va, taddr + c * 32, doc0 + c * 32);
                    tmem_ld_wait();
                    if (c + 2 < COLS / 32) tmem_ld32(taddr + (c + 2) * 32, va);
                    filter(vb, taddr + (c + 1) * 32, doc0 + (c + 1) * 32);
                    tmem_ld_wait();
                }
                fence_before();  // the accumulator has been read: hand it back to the issuer
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
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
                    if (c > k) { mma::select_row(row, c, k, hist, lane); c = k; }
                    __syncwarp();
                    uint64_t *dst = p.out + (part * p.nq + qq) * k;
                    for (int e = lane; e < k; e += 32) dst[e] = e < c ? __ldcg(row + e) : KEY_INF;
                }
                __syncwarp();
            }
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
    } else if (warp < EPI_WARPS + PROD_WARPS) {
        // ================================ producers ================================
        reg_dec<PROD_REGS>();
        const int pw = warp - EPI_WARPS;
        const int qd = lane >> 3, d = (lane >> 2) & 1, gg = lane & 3;
        const int kb = qd % C, doc_in_it = 2 * (qd / C) + d, g = 4 * kb + gg;
        const unsigned char *db = reinterpret_cast<const unsigned char *>(p.db);
        const uint32_t n_pad32 = static_cast<uint32_t>(p.n_pad);
        auto load_stage = [&](uint4 (&r)[ITW], int sd) {
#pragma unroll
            for (int it = 0; it < ITW; ++it) {
                const uint32_t row = static_cast<uint32_t>(sd) * STAGE_DOCS + (it * PROD_WARPS + pw) * DPI + doc_in_it;
                r[it] = row < n_pad32 ? __ldg(reinterpret_cast<const uint4 *>(db + static_cast<int64_t>(row) * ROW_BYTES + g * 16))
                                      : make_uint4(0u, 0u, 0u, 0u);
            }
        };
        auto store_stage = [&](const uint4 (&r)[ITW], int slot) {
            unsigned char *stage = sB + static_cast<size_t>(slot) * B_STAGE + kb * (STAGE_DOCS * 128);
#pragma unroll
            for (int it = 0; it < ITW; ++it) {
                const int row = (it * PROD_WARPS + pw) * DPI + doc_in_it;
                unsigned char *rowp = stage + (row >> 3) * 1024 + (row & 7) * 128;
                const uint4 w = r[it];
                *reinterpret_cast<uint4 *>(rowp + (((2 * gg) ^ (row & 7)) << 4)) =
                    make_uint4(w.x & 0x0F0F0F0Fu, (w.x >> 4) & 0x0F0F0F0Fu, w.y & 0x0F0F0F0Fu, (w.y >> 4) & 0x0F0F0F0Fu);
                *reinterpret_cast<uint4 *>(rowp + (((2 * gg + 1) ^ (row & 7)) << 4)) =
                    make_uint4(w.z & 0x0F0F0F0Fu, (w.z >> 4) & 0x0F0F0F0Fu, w.w & 0x0F0F0F0Fu, (w.w >> 4) & 0x0F0F0F0Fu);
            }
        };
        while (sg.next()) {
            stage_queries(sg.gr);
            cta_sync();
            Ring rb{static_cast<int>(s_run % NS), ((s_run / NS) & 1u) ^ 1u};  // "empty" waits start on the completed phase
            auto publish = [&](const uint4 (&r)[ITW]) {
                mbar_wait(&b_empty[rb.idx], rb.phase);
                store_stage(r, rb.idx);
                fence_async_smem();  // generic-proxy stores -> visible to the tensor core's async proxy
                __syncwarp();
                if (lane == 0) mbar_arrive(&b_full[rb.idx]);
                rb.advance(NS);
            };
            uint4 ra[ITW], rbuf[ITW];
            load_stage(ra, sg.sd0);
            if (sg.cnt > 1) load_stage(rbuf, sg.sd0 + 1);
            for (int i = 0; i < sg.cnt; i += 2) {
                publish(ra);
                if (i + 2 < sg.cnt) load_stage(ra, sg.sd0 + i + 2);
                if (i + 1 < sg.cnt) {
                    publish(rbuf);
                    if (i + 3 < sg.cnt) load_stage(rbuf, sg.sd0 + i + 3);
                }
            }
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
    } else {
        // ================================ MMA issuer (+ three idle warps) ================================
        reg_dec<MMA_REGS>();
        const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
        while (sg.next()) {
            stage_queries(sg.gr);
            cta_sync();
            if (warp == MMA_WARP && lane == 0) {
                Ring rb{static_cast<int>(s_run % NS), (s_run / NS) & 1u};
                for (int i = 0; i < sg.cnt; ++i) {
                    mbar_wait(&b_full[rb.idx], rb.phase);
                    fence_after();
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const uint32_t u = (s_run + i) * MT + mt;
                        const uint32_t buf = u & (ACC_BUFS - 1), use = u / ACC_BUFS;
                        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
                        fence_after();
#pragma unroll
                        for (int ks = 0; ks < KSTEPS; ++ks) {
                            const uint64_t ad = make_desc(a_base + mt * A_TILE + (ks >> 2) * (128 * 128) + (ks & 3) * 32);
                            const uint64_t bd = make_desc(b_base + rb.idx * B_STAGE + (ks >> 2) * (STAGE_DOCS * 128) + (ks & 3) * 32);
                            umma_i8(tmem + buf * STAGE_DOCS, ad, bd, ks > 0 ? 1u : 0u);
                        }
                        umma_commit(&acc_full[buf]);
                    }
                    umma_commit(&b_empty[rb.idx]);
                    rb.advance(NS);
                }
            }
            __syncwarp();
            s_run += static_cast<uint32_t>(sg.cnt);
            cta_sync();
        }
    }
    fence_before();
    cta_sync();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace umma
