// xfbq_coop.cuh -- single-launch search for small batches (<= 16 queries), included by xfbq_b200.cu.
//
// The mma.sync scan of xfbq_mma.cuh is HBM-bound for <= 16 queries (a 10M x 256 scan takes 0.23 ms), but a search used to be
// ten launches around it -- query preparation (2), threshold seeding (4), the scan, two merge levels -- whose kernels and
// launch gaps added 0.13 ms.  This kernel is the whole search as ONE cooperative launch (one persistent CTA per SM, grid-wide
// barriers between the phases):
//   1  CTA r < 16 turns query row r into MMA A fragments (s8 weights 2y - Aq) and Dq; everybody zeroes the histograms; the
//      TMA ring already starts filling with the CTA's first document stages
//   2  every warp scores SEED_TILES tiles of documents spread over the whole database (2 368 warps x 2 x 16 documents: a
//      75k-document sample) and bumps one bin per score of a fixed-frame histogram over the full score range
//   3  CTA r reads query r's threshold off its histogram: the highest bin whose suffix count reaches k proves that k real
//      documents score at least the bin's lower edge
//   4  the scan: TMA ring -> registers -> IMMA -> sign test against the row thresholds -> per-warp candidate lists; every
//      candidate also bumps a 256-bin histogram of its query measured from the seeded threshold, a few warps per CTA turn
//      those into tighter thresholds ("bins >= b hold >= k candidates") shared through theta_g, which every warp polls
//   5  CTA r merges query r's lists where they lie (bounded by the final threshold) and writes the k best keys.
// Results are exact whatever the thresholds do: they are lower bounds of the k-th best score proven by counted documents.
#pragma once
#include <cooperative_groups.h>
#include <limits.h>

namespace coop {

namespace cg = cooperative_groups;
using mma::imma;
using mma::mbar_arrive;
using mma::mbar_arrive_expect_tx;
using mma::mbar_init;
using mma::mbar_test;
using mma::mbar_wait;
using mma::Ring;
using mma::TAU_OPEN;
using mma::tma_bulk_g2s;

constexpr int WARPS = 16;
constexpr int SEED_BINS = 4096;   // fixed frame over the whole score range [-R, R], R = dim * Ad * Aq
constexpr int SEED_TILES = 2;     // sample tiles per warp
constexpr int CAND_BINS = 256;    // candidate histogram, measured from the seeded threshold (umma::hist_bound)

struct Params {
    const void *nib;           // nibble layout
    int64_t n, n_pad, row_offset;
    const uint32_t *q;         // query layout [nq][wq][4C] (quantized queries), or nullptr:
    const void *xq;            // float queries [nq][ldq] (float32, or float64 when xq_f64), quantized in phase 1 exactly as
    int xq_f64;                // quantize_queries_kernel does (quant.py:138-148 after bitplane.py:214-222)
    int64_t ldq;
    double scale;
    unsigned long long *nonfinite;  // += non-finite scaled query values (the reference raises, quant.py:142-143); such a row
    int *row_bad;                   // [16] is flagged here and answered with empty keys
    int nq, wq, wd, dim;
    uint32_t *qop;             // [4C k-steps][32 lanes][4] A fragments of the 16-row tile (written in phase 1)
    int32_t *qconst;           // [16] Dq
    uint32_t *shist;           // [16][SEED_BINS]
    int32_t *theta_g;          // [16] shared thresholds (accumulator domain)
    int32_t *theta0;           // [16] seeded thresholds: origin of the candidate histogram
    uint32_t *chist;           // [16][CAND_BINS]
    uint64_t *lists;           // [grid * WARPS][16][cap]
    int *counts;               // [16][grid * WARPS] list lengths (row-major by query: coalesced for the merging CTA)
    uint64_t *final_list;      // [16][final_cap] list entries the FINAL thresholds still admit, forwarded by every warp after the scan
    unsigned *final_cnt;       // [16] their number (may exceed final_cap: then the merging CTA reads the lists themselves)
    int final_cap;
    uint64_t *keys_out;        // [nq][k]
    int64_t stages;            // stages of WARPS * TILE documents
    int64_t seed_tile_stride;  // sample tile i of the grid is tile i * seed_tile_stride of the database
    int k, cap, RR;
    int seed_shift, seed_offset;  // bin = (acc + seed_offset) >> seed_shift
    int hist_shift;               // candidate bins of width 1 << hist_shift
    int merge_B;                  // keys of the final merge buffer (power of two)
    // k_select in the same launch (search.py:206-216): the scan prunes `extra` score units below the thresholds, so the lists
    // hold every row with distance <= (k-th distance + extra); the merge counts them per query (and lists their ids) unless a
    // list had to be cut during the scan (*inexact != 0: the caller falls back to the separate gather pass)
    int extra;
    unsigned long long *cand_count;   // [nq] or nullptr (feature off)
    int64_t *cand_ids;                // [nq][cand_cap] or nullptr
    int64_t cand_cap;
    int *inexact;                     // [1]
    unsigned long long *prof;     // optional [8 + 2 * grid] phase time stamps (ns, xfbq_debug_profile), else nullptr
};
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Query row -> A fragments + Dq (the body of mma::prep_queries_kernel for one row of tile 0); one warp.  The codes come from
// the quantized query planes, or straight from the float row.
__device__ __forceinline__ void prep_row(const Params &p, int row, int C, int lane) {
    const int W = 4 * C;
    const int Aq = (1 << p.wq) - 1, Ad = (1 << p.wd) - 1;
    const double half = static_cast<double>(1 << (p.wq - 1));
    unsigned long long bad = 0;
    int sy = 0;
    for (int ow = lane; ow < 32 * C; ow += 32) {
        const int hi = ow & 1, t = (ow >> 1) & 3, s = ow >> 3;
        const int h = s >> 2, e = s & 3;
        uint32_t packed = 0;
        if (row < p.nq) {
            const int word = C * t + h;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int bit = 8 * j + e + 4 * hi;
                const int d = 32 * word + bit;
                if (d < p.dim) {
                    int y = 0;
                    if (p.q) {
                        for (int jq = 0; jq < p.wq; ++jq) y |= static_cast<int>((p.q[(static_cast<int64_t>(row) * p.wq + jq) * W + word] >> bit) & 1u) << jq;
                    } else if (p.xq_f64) {
                        y = static_cast<int>(quantize_one<double>(static_cast<const double *>(p.xq)[row * p.ldq + d], p.scale, half, bad));
                    } else {
                        y = static_cast<int>(quantize_one<float>(static_cast<const float *>(p.xq)[row * p.ldq + d], p.scale, half, bad));
                    }
                    sy += y;
                    packed |= (static_cast<uint32_t>(2 * y - Aq) & 0xFFu) << (8 * j);
                }
            }
        }
        p.qop[((s * 32) + (row & 7) * 4 + t) * 4 + (row >> 3) + 2 * hi] = packed;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
        p.qconst[row] = (row < p.nq) ? Ad * sy : 0;
        p.row_bad[row] = bad ? 1 : 0;
        if (bad && p.nonfinite) atomicAdd(p.nonfinite, bad);
    }
}

template <int C>
__global__ void __launch_bounds__(WARPS * 32, 1) search_kernel(const Params p) {
    constexpr int NT = C <= 2 ? 2 : 1;
    constexpr int KS = 4 * C;
    constexpr int TILE = 8 * NT;
    constexpr int WPL = NT * C * 8;
    constexpr int STAGE_DOCS = WARPS * TILE;
    constexpr int ROW_BYTES = 64 * C;
    constexpr int RAW_STAGE_BYTES = STAGE_DOCS * ROW_BYTES;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ int s_pre[148 * WARPS + 1 + 64];  // final merge: list-length prefix sums (grid <= 148 + slack)
    __shared__ uint32_t s_wsum[WARPS];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int RR = p.RR;
    const mma::SmemLayout L = mma::smem_layout(RAW_STAGE_BYTES, 0, RR, 0, p.cap, WARPS);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + L.bar_off);
    uint64_t *raw_full = bars, *raw_empty = bars + RR;

    // ---- this CTA's document stages
    const int64_t T = p.stages, G = gridDim.x;
    const int64_t lin_begin = static_cast<int64_t>(blockIdx.x) * T / G, lin_end = (static_cast<int64_t>(blockIdx.x) + 1) * T / G;
    const int S = static_cast<int>(lin_end - lin_begin);
    if (threadIdx.x == 0) {
        for (int i = 0; i < RR; ++i) { mbar_init(&raw_full[i], 1); mbar_init(&raw_empty[i], WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t db_bytes = p.n_pad * static_cast<int64_t>(ROW_BYTES);
    Ring is_ring{0, 1u};
    int64_t is_sd = lin_begin;
    int issued = 0;
    auto pump = [&]() {  // thread 0 refills every raw-ring slot that all warps have released
        if (threadIdx.x != 0) return;
        while (issued < S && mbar_test(&raw_empty[is_ring.idx], is_ring.phase)) {
            const int64_t off = is_sd * RAW_STAGE_BYTES;
            int64_t bytes = db_bytes - off;
            if (bytes > RAW_STAGE_BYTES) bytes = RAW_STAGE_BYTES;
            mbar_arrive_expect_tx(&raw_full[is_ring.idx], static_cast<uint32_t>(bytes));
            tma_bulk_g2s(smem_raw + L.raw_off + static_cast<size_t>(is_ring.idx) * RAW_STAGE_BYTES,
                         reinterpret_cast<const unsigned char *>(p.nib) + off, static_cast<uint32_t>(bytes), &raw_full[is_ring.idx]);
            is_ring.advance(RR);
            ++is_sd;
            ++issued;
        }
    };
    auto wait_bar = [&](uint64_t *bar, uint32_t parity) {
        if (warp == 0) {
            while (!mbar_test(bar, parity)) pump();
        } else {
            mbar_wait(bar, parity);
        }
    };
    pump();  // the first stages stream in while the queries are prepared and the thresholds seeded
    auto stamp = [&](int i) { if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) p.prof[i] = now_ns(); };
    stamp(0);

    // ================================ phase 1: query operand, cleared histograms ================================
    {
        const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x, gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
        for (int64_t i = gtid; i < 16 * SEED_BINS; i += gthreads) p.shist[i] = 0u;
        for (int64_t i = gtid; i < 16 * CAND_BINS; i += gthreads) p.chist[i] = 0u;
        if (gtid < 16) { p.theta_g[gtid] = TAU_OPEN; p.theta0[gtid] = TAU_OPEN; }
        if (gtid == 0 && p.inexact) *p.inexact = 0;
        if (gtid < 16) p.final_cnt[gtid] = 0u;
        for (int row = blockIdx.x; row < 16; row += gridDim.x)
            if (warp == 0) prep_row(p, row, C, lane);
    }
    __threadfence();
    grid.sync();
    stamp(1);

    // ---- per-warp state: lane (g, t) of the MMA layout; lane l < 16 also owns query row l
    const int g = lane >> 2, t = lane & 3;
    uint32_t a[KS][4];
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(p.qop) + s * 32 + lane);
        a[s][0] = v.x; a[s][1] = v.y; a[s][2] = v.z; a[s][3] = v.w;
    }
    const bool row_valid = lane < 16 && lane < p.nq;
    static_assert(148 * WARPS < 5 * WARPS * 32, "list-length prefix: five lists per thread");
    const int my_dq = row_valid ? __ldcg(p.qconst + lane) : 0;
    const uint32_t n_docs = static_cast<uint32_t>(p.n);
    const int gw = blockIdx.x * WARPS + warp;
    uint64_t *lists = p.lists + static_cast<int64_t>(gw) * 16 * static_cast<int64_t>(p.cap);
    int *cnt_s = reinterpret_cast<int *>(smem_raw + L.cnt_off) + warp * 32;
    const bool small_lists = p.cap <= mma::SORT_CAP_MAX;
    uint64_t *scratch = reinterpret_cast<uint64_t *>(smem_raw + L.scratch_off) + static_cast<size_t>(warp) * p.cap;
    int *hist = reinterpret_cast<int *>(smem_raw + L.scratch_off) + warp * 256;

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
    // scores of one tile, biased by -tau of the rows (bias0 / bias1: rows g / g + 8)
    auto scores = [&](const uint32_t (&bw)[WPL], int bias0, int bias1, int (&c)[NT][4]) {
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const uint32_t b0 = bw[(nt * C + (s2 >> 2)) * 8 + 2 * (s2 & 3)];
                const uint32_t b1 = bw[(nt * C + (s2 >> 2)) * 8 + 2 * (s2 & 3) + 1];
                if (s2 == 0) imma(c[nt], a[s2], b0, b1, bias0, bias0, bias1, bias1);
                else imma(c[nt], a[s2], b0, b1, c[nt][0], c[nt][1], c[nt][2], c[nt][3]);
            }
    };

    // ================================ phase 2: sample histogram ================================
    // Every warp scores SEED_TILES spread tiles; each lane then counts only its BEST sample score of a row (four lanes
    // share a row: 4 of the warp's 32 sample documents per row).  Counting a subset is safe -- the bins still count real,
    // distinct documents -- and nearly free of loss (a warp's 32 documents rarely hold more than a few of the sample's
    // k best), while counting every score made 75k atomics fight over the few dozen bins around the mean (25-40 us).
    {
        const uint4 *nib = reinterpret_cast<const uint4 *>(p.nib);
        uint4 nw[SEED_TILES][NT][C];
        int64_t doc0s[SEED_TILES];
#pragma unroll
        for (int st = 0; st < SEED_TILES; ++st) {
            const int64_t tile = (static_cast<int64_t>(gw) * SEED_TILES + st) * p.seed_tile_stride;
            doc0s[st] = tile * TILE;
            const bool inside = doc0s[st] + TILE <= p.n_pad;  // warp-uniform
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < C; ++h)
                    nw[st][nt][h] = inside ? __ldg(nib + (doc0s[st] + 8 * nt + g) * (4 * C) + C * t + h) : make_uint4(0u, 0u, 0u, 0u);
        }
        int best0 = INT_MIN, best1 = INT_MIN;  // rows g, g + 8
#pragma unroll
        for (int st = 0; st < SEED_TILES; ++st) {
            if (doc0s[st] + TILE > p.n_pad) continue;
            uint32_t bw[WPL];
            nibbles_to_fragments(nw[st], bw);
            int c[NT][4];
            scores(bw, 0, 0, c);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t doc = doc0s[st] + 8 * nt + 2 * t + (j & 1);
                    if (doc < p.n) {
                        if (j >> 1) best1 = max(best1, c[nt][j]); else best0 = max(best0, c[nt][j]);
                    }
                }
        }
        if (g < p.nq && best0 != INT_MIN)
            atomicAdd(p.shist + g * SEED_BINS + min(max((best0 + p.seed_offset) >> p.seed_shift, 0), SEED_BINS - 1), 1u);
        if (g + 8 < p.nq && best1 != INT_MIN)
            atomicAdd(p.shist + (g + 8) * SEED_BINS + min(max((best1 + p.seed_offset) >> p.seed_shift, 0), SEED_BINS - 1), 1u);
    }
    __threadfence();
    grid.sync();
    stamp(2);

    // ================================ phase 3: thresholds off the sample histograms ================================
    for (int r = blockIdx.x; r < p.nq; r += gridDim.x) {
        // thread t owns bins [8t, 8t + 8); suffix counts over the block
        const uint4 *bins = reinterpret_cast<const uint4 *>(p.shist + r * SEED_BINS) + 2 * threadIdx.x;
        const uint4 lo = __ldcg(bins), hi = __ldcg(bins + 1);
        const uint32_t cb[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        uint32_t s = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) s += cb[e];
        uint32_t suf = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_down_sync(0xffffffffu, suf, o);
            if (lane + o < 32) suf += v;
        }
        __syncthreads();
        if (lane == 0) s_wsum[warp] = suf;
        __syncthreads();
        for (int w = warp + 1; w < WARPS; ++w) suf += s_wsum[w];
        const uint32_t kk = static_cast<uint32_t>(p.k);
        if (suf >= kk && suf - s < kk) {  // exactly one thread when the sample holds >= k documents
            uint32_t acc = suf - s;
            int b = -1;
#pragma unroll
            for (int e = 7; e >= 0; --e) {
                acc += cb[e];
                if (b < 0 && acc >= kk) b = 8 * static_cast<int>(threadIdx.x) + e;
            }
            const int th = (b << p.seed_shift) - p.seed_offset;  // every score of bin b is >= its lower edge
            p.theta0[r] = th;
            p.theta_g[r] = th;
        }
    }
    __threadfence();
    grid.sync();
    stamp(3);

    // ================================ phase 4: the scan ================================
    int my_tau = row_valid ? max(TAU_OPEN, __ldcg(p.theta_g + lane)) : 1;   // no query: acc = 0 < 1
    const int my_th0 = row_valid ? __ldcg(p.theta0 + lane) : 0;
    __syncwarp();
    cnt_s[lane] = 0;
    __syncwarp();
    // a row passes a score when acc >= tau - extra (extra > 0 only for k_select's candidate slack); rows without a query never pass
    auto prune_of = [&](int tau) { return row_valid ? max(TAU_OPEN, tau - p.extra) : 1; };
    int negtau0 = -__shfl_sync(0xffffffffu, prune_of(my_tau), g), negtau1 = -__shfl_sync(0xffffffffu, prune_of(my_tau), g + 8);

    const int dq0 = __shfl_sync(0xffffffffu, my_dq, g), dq1 = __shfl_sync(0xffffffffu, my_dq, g + 8);
    const int th00 = __shfl_sync(0xffffffffu, my_th0, g), th01 = __shfl_sync(0xffffffffu, my_th0, g + 8);

    auto push = [&](const int (&v)[4], uint32_t doc_a) {  // (v0, v1): row g, docs doc_a, doc_a + 1; (v2, v3): row g + 8
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t doc = doc_a + (j & 1);
            if (v[j] >= 0 && doc < n_docs) {
                const int row = g + 8 * (j >> 1);
                const int acc = v[j] - (j >> 1 ? negtau1 : negtau0);        // the raw score
                const uint32_t dist = static_cast<uint32_t>((j >> 1 ? dq1 : dq0) - acc);
                const int pos = atomicAdd(&cnt_s[row], 1);
                lists[row * p.cap + pos] = (static_cast<uint64_t>(dist) << 32) | (static_cast<uint64_t>(p.row_offset) + doc);
                const int th0 = j >> 1 ? th01 : th00;
                if (th0 > TAU_OPEN)
                    atomicAdd(p.chist + row * CAND_BINS + min(max((acc - th0) >> p.hist_shift, 0), CAND_BINS - 1), 1u);
            }
        }
    };
    auto process = [&](const uint32_t (&bw)[WPL], uint32_t doc0) {
        int c[NT][4];
        scores(bw, negtau0, negtau1, c);
        int all = -1;
        int pm[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            pm[nt] = (c[nt][0] & c[nt][1]) & (c[nt][2] & c[nt][3]);
            all &= pm[nt];
        }
        if (__any_sync(0xffffffffu, all >= 0)) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
                if (pm[nt] >= 0) push(c[nt], doc0 + 8 * nt + 2 * t);
            __syncwarp();
            unsigned need = __ballot_sync(0xffffffffu, lane < 16 && cnt_s[lane] > p.cap - TILE);
            while (need) {  // a list the next tile could overflow: keep its k best, tighten its row's threshold
                const int ql = __ffs(need) - 1;
                need &= need - 1;
                const int nv = small_lists ? mma::compact_row_sorted(lists + ql * p.cap, scratch, &cnt_s[ql], p.k, ql, lane, my_dq, &my_tau)
                                           : mma::compact_row(lists + ql * p.cap, hist, &cnt_s[ql], p.k, ql, lane, my_dq, &my_tau);
                negtau0 = -__shfl_sync(0xffffffffu, prune_of(my_tau), g);
                negtau1 = -__shfl_sync(0xffffffffu, prune_of(my_tau), g + 8);
                if (lane == ql) {
                    atomicMax(p.theta_g + ql, -nv);
                    if (p.inexact) *p.inexact = 1;   // the list was cut to its k best: it no longer holds every candidate
                }
            }
        }
    };

    const uint32_t n_pad32 = static_cast<uint32_t>(p.n_pad);
    Ring rf{0, 0u};
    int tg_next = TAU_OPEN;
    for (int ci = 0; ci < S; ++ci) {
        uint4 nw[NT][C];
        uint32_t bw[WPL];
        if ((ci & 7) == 0 && row_valid) tg_next = __ldcg(p.theta_g + lane);  // fetched eight stages ahead of its use
        wait_bar(&raw_full[rf.idx], rf.phase);
        {
            const uint4 *raw = reinterpret_cast<const uint4 *>(smem_raw + L.raw_off + static_cast<size_t>(rf.idx) * RAW_STAGE_BYTES);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < C; ++h) nw[nt][h] = raw[(warp * TILE + 8 * nt + g) * (4 * C) + C * t + h];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&raw_empty[rf.idx]);
        rf.advance(RR);
        pump();
        const uint32_t doc0 = (static_cast<uint32_t>(lin_begin + ci) * WARPS + warp) * TILE;
        if (doc0 + TILE <= n_pad32) {
            nibbles_to_fragments(nw, bw);
            process(bw, doc0);
        }
        if ((ci & 7) == 7) {  // adopt what the other warps and CTAs have proven for our rows
            const int tnew = max(my_tau, tg_next);
            if (__any_sync(0xffffffffu, tnew != my_tau)) {
                my_tau = tnew;
                negtau0 = -__shfl_sync(0xffffffffu, prune_of(my_tau), g);
                negtau1 = -__shfl_sync(0xffffffffu, prune_of(my_tau), g + 8);
            }
        }
        // One warp of the CTA per 16 stages (per 64 once the thresholds have settled) turns one query's candidate histogram
        // into a bound for everybody.  The two L2 round trips stall that warp for ~2 us, which the ring's slack absorbs; with
        // 148 CTAs taking turns every query is refreshed every fraction of a microsecond.
        {
            const int period_mask = ci < 128 ? 15 : 63;
            if ((ci & period_mask) == period_mask && warp == ((ci >> 4) & (WARPS - 1))) {
                const int r = static_cast<int>((blockIdx.x + static_cast<unsigned>(ci >> 4)) % static_cast<unsigned>(p.nq));
                const int th0 = __shfl_sync(0xffffffffu, my_th0, r);
                if (th0 > TAU_OPEN) {
                    const uint4 *bins = reinterpret_cast<const uint4 *>(p.chist + r * CAND_BINS) + 2 * lane;
                    const uint4 lo = __ldcg(bins), hi = __ldcg(bins + 1);
                    const int b = umma::hist_bound(lo, hi, p.k, lane);
                    if (b > 0 && lane == 0) atomicMax(p.theta_g + r, th0 + (b << p.hist_shift));
                }
            }
        }
    }

    // ================================ phase 5: merge the lists where they lie ================================
    __syncwarp();
    if (p.prof && threadIdx.x == 0) p.prof[8 + blockIdx.x] = now_ns();  // this CTA's scan is done
    if (lane < 16) p.counts[lane * (static_cast<int>(gridDim.x) * WARPS) + gw] = cnt_s[lane];  // [row][list]: coalesced for the merging CTA
    __threadfence();
    grid.sync();
    stamp(4);
    // ---- 5a: the thresholds are final now; every warp forwards the entries of its own lists that they still admit (about k per
    // query in all, against ~20 k entries at k = 1000) to one compact list per query, so that the merging CTA sorts a handful
    // of keys instead of walking 2 368 lists (merge 85 -> see profiles, 12.5M x 512, k = 1000)
    {
        const int tgf = row_valid ? __ldcg(p.theta_g + lane) : TAU_OPEN;
        for (int r = 0; r < p.nq; ++r) {
            const int cnt = cnt_s[r];
            const int tg = __shfl_sync(0xffffffffu, tgf, r), dq = __shfl_sync(0xffffffffu, my_dq, r);
            const long long limit = tg > TAU_OPEN ? static_cast<long long>(dq) - tg + p.extra : 0x7FFFFFFFll;
            for (int e0 = 0; e0 < cnt; e0 += 32) {
                const int e = e0 + lane;
                const uint64_t key = e < cnt ? __ldcg(lists + r * p.cap + e) : KEY_INF;
                const bool keep = key != KEY_INF && static_cast<long long>(key >> 32) <= limit;
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (m) {
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(p.final_cnt + r, static_cast<unsigned>(__popc(m)));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
                    if (keep && pos < static_cast<unsigned>(p.final_cap)) p.final_list[static_cast<int64_t>(r) * p.final_cap + pos] = key;
                }
            }
        }
    }
    __threadfence();
    grid.sync();
    for (int r = blockIdx.x; r < p.nq; r += gridDim.x) {
        const int parts = static_cast<int>(gridDim.x) * WARPS;
        __syncthreads();
        if (__ldcg(p.row_bad + r)) {  // a non-finite query: no answer (block-uniform)
            for (int i = threadIdx.x; i < p.k; i += blockDim.x) p.keys_out[static_cast<int64_t>(r) * p.k + i] = KEY_INF;
            continue;
        }
        const unsigned nfin = __ldcg(p.final_cnt + r);
        if (nfin <= static_cast<unsigned>(p.final_cap) && static_cast<int>(nfin) + static_cast<int>(blockDim.x) <= p.merge_B) {
            // ---- 5b: sort the compact list, write the k best; k_select's candidates are counted from it as well
            const uint64_t *fl = p.final_list + static_cast<int64_t>(r) * p.final_cap;
            merge_bounded_block(reinterpret_cast<uint64_t *>(smem_raw), p.merge_B, p.k, static_cast<int64_t>(nfin), 0x7FFFFFFFll,
                                [&](int64_t e) -> uint64_t { return __ldcg(fl + e); }, p.keys_out + static_cast<int64_t>(r) * p.k);
            if (p.cand_count) {
                __syncthreads();
                const int valid = static_cast<int>(nfin) < p.k ? static_cast<int>(nfin) : p.k;
                const long long thr = valid > 0 ? static_cast<long long>(__ldcg(p.keys_out + static_cast<int64_t>(r) * p.k + valid - 1) >> 32) + p.extra : -1;
                if (threadIdx.x == 0) p.cand_count[r] = 0ull;
                __syncthreads();
                for (unsigned e0 = 0; e0 < nfin; e0 += blockDim.x) {
                    const unsigned e = e0 + threadIdx.x;
                    const uint64_t key = e < nfin ? __ldcg(fl + e) : KEY_INF;
                    const bool hit = key != KEY_INF && static_cast<long long>(key >> 32) <= thr;
                    const unsigned m = __ballot_sync(0xffffffffu, hit);
                    if (m) {
                        unsigned long long base = 0;
                        if (lane == 0) base = atomicAdd(p.cand_count + r, static_cast<unsigned long long>(__popc(m)));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        const int64_t pos = static_cast<int64_t>(base) + __popc(m & ((1u << lane) - 1u));
                        if (hit && p.cand_ids && pos < p.cand_cap) p.cand_ids[static_cast<int64_t>(r) * p.cand_cap + pos] = static_cast<int64_t>(key & 0xFFFFFFFFull);
                    }
                }
            }
            if (p.prof && r == 0 && threadIdx.x == 0) { p.prof[5] = now_ns(); p.prof[6] = static_cast<unsigned long long>(nfin); }
            continue;
        }
        // ---- fallback (more admitted entries than the compact list holds: heavy ties): walk the lists themselves
        {   // s_pre[i] = entries in lists < i: thread t sums its run of PER lists, a block scan over the 512 partial sums follows
            constexpr int PER = (148 * WARPS + WARPS * 32 - 1) / (WARPS * 32);
            int len[PER], sum = 0;
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int part = static_cast<int>(threadIdx.x) * PER + e;
                len[e] = part < parts ? __ldcg(p.counts + r * parts + part) : 0;
                sum += len[e];
            }
            int inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            if (lane == 31) s_wsum[warp] = static_cast<uint32_t>(inc);
            __syncthreads();
            int base = inc - sum;
            for (int w = 0; w < warp; ++w) base += static_cast<int>(s_wsum[w]);
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int part = static_cast<int>(threadIdx.x) * PER + e;
                if (part <= parts) s_pre[part] = base;
                base += len[e];
            }
        }
        __syncthreads();
        const int tg = __ldcg(p.theta_g + r);
        const long long limit = tg > TAU_OPEN ? static_cast<long long>(__ldcg(p.qconst + r)) - tg : 0x7FFFFFFFll;
        merge_bounded_block(reinterpret_cast<uint64_t *>(smem_raw), p.merge_B, p.k, s_pre[parts], limit, [&](int64_t e) -> uint64_t {
            const int part = find_part(s_pre, parts, static_cast<int>(e));
            return __ldcg(p.lists + (static_cast<int64_t>(part) * 16 + r) * p.cap + (e - s_pre[part]));
        }, p.keys_out + static_cast<int64_t>(r) * p.k);
        if (p.cand_count) {  // every list entry within `extra` of the k-th distance (the k best keys have just been written)
            __syncthreads();
            const int total = s_pre[parts];
            const int valid = total < p.k ? total : p.k;
            const long long thr = valid > 0 ? static_cast<long long>(__ldcg(p.keys_out + static_cast<int64_t>(r) * p.k + valid - 1) >> 32) + p.extra : -1;
            if (threadIdx.x == 0) p.cand_count[r] = 0ull;
            __syncthreads();
            for (int e0 = 0; e0 < total; e0 += blockDim.x) {
                const int e = e0 + threadIdx.x;
                uint64_t key = KEY_INF;
                if (e < total) {
                    const int part = find_part(s_pre, parts, e);
                    key = __ldcg(p.lists + (static_cast<int64_t>(part) * 16 + r) * p.cap + (e - s_pre[part]));
                }
                const bool hit = key != KEY_INF && static_cast<long long>(key >> 32) <= thr;
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (m) {
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(p.cand_count + r, static_cast<unsigned long long>(__popc(m)));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    const int64_t pos = static_cast<int64_t>(base) + __popc(m & ((1u << lane) - 1u));
                    if (hit && p.cand_ids && pos < p.cand_cap) p.cand_ids[static_cast<int64_t>(r) * p.cand_cap + pos] = static_cast<int64_t>(key & 0xFFFFFFFFull);
                }
            }
        }
        if (p.prof && r == 0 && threadIdx.x == 0) { p.prof[5] = now_ns(); p.prof[6] = static_cast<unsigned long long>(s_pre[parts]); }
    }
}

}  // namespace coop
