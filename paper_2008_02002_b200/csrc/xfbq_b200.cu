// xfbq_b200.cu -- hand-written sm_100a kernels + C ABI for the XFBQ hot path.
//
// quantize -> bit-plane pack -> XOR/POPC scan with fused top-K -> merge.
// See include/xfbq_b200.h for the ABI contract and the device layouts, DESIGN.md for
// the roofline of each kernel.  Reference citations are paths under
// /root/reference/pkg/src/xfbq.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
// (no --use_fast_math: the quantizer depends on IEEE float64 and on denormal inputs).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <unistd.h>

#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>

extern char **environ;

#include "../../include/xfbq_b200.h"

#define XFBQ_API extern "C" __attribute__((visibility("default")))

namespace {

constexpr uint64_t KEY_INF = 0xFFFFFFFFFFFFFFFFull;
constexpr int SCAN_THREADS = 256;  // 8 warps = 8 bundles = 256 documents per step
constexpr int SCAN_WARPS = SCAN_THREADS / 32;

thread_local char g_err[512] = "";
// optional device timing of the main scan kernel (xfbq_set_timing): events live per host thread
thread_local bool g_timing = false;
// a ring of event pairs: every timed launch since xfbq_set_timing(1) takes the next pair (the last TIMING_PAIRS are kept),
// so a bench reads the MEAN launch time of its timed region, not the last launch only
constexpr int TIMING_PAIRS = 64;
thread_local cudaEvent_t g_evs[TIMING_PAIRS][2] = {};
thread_local int g_ev_count = 0;   // timed launches recorded since timing was switched on
std::atomic<int64_t> g_launches{0};
thread_local unsigned long long *g_prof = nullptr;
thread_local int g_hist_shift = 2;  // bin width of the tcgen05 engine's global candidate histogram (set per search from the distance range)  // debug: device buffer for the tcgen05 engine's wait counters

void timing_begin(cudaStream_t st) { cudaEventRecord(g_evs[g_ev_count % TIMING_PAIRS][0], st); }
void timing_end(cudaStream_t st) { cudaEventRecord(g_evs[g_ev_count % TIMING_PAIRS][1], st); ++g_ev_count; }

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return XFBQ_OK;
}

inline int64_t chunks128(int64_t dim) { return (dim + 127) / 128; }
inline int64_t bundles_of(int64_t n) { return (n + 31) / 32; }
inline bool width_ok(int w) { return w >= 1 && w <= XFBQ_MAX_WIDTH; }

struct DeviceInfo {
    int sms = 0;
    int smem_optin = 0;
};

int device_info(DeviceInfo *info) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    static thread_local int cached_dev = -1;
    static thread_local DeviceInfo cached;
    if (cached_dev != dev) {
        e = cudaDeviceGetAttribute(&cached.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaDeviceGetAttribute(&cached.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
        cached_dev = dev;
    }
    *info = cached;
    return XFBQ_OK;
}

// ----------------------------------------------------------------------------------------------
// Quantizer (quant.py:138-148 after bitplane.py:229-232): float64 arithmetic, exactly
//   t = floor((double(x) * scale) * 2^(w-1));  t = clamp(t, -2^(w-1), 2^(w-1)-1);  code = 2^(w-1)-1-t
// which equals (hi - clip(2*floor(..)+1, -hi, hi)) / 2 with hi = 2^w - 1.
// ----------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ unsigned quantize_one(T x, double scale, double half, unsigned long long &bad) {
    double v = static_cast<double>(x) * scale;      // bitplane.py:232
    if (!isfinite(v)) { ++bad; return 0u; }         // quant.py:142-143
    double t = floor(v * half);                     // quant.py:146 (overflow to +-inf saturates below)
    t = fmin(fmax(t, -half), half - 1.0);           // quant.py:147 clip
    return static_cast<unsigned>(static_cast<int>(half) - 1 - static_cast<int>(t));
}

// One warp packs one bundle (32 documents) chunk by chunk: lanes read 32 consecutive
// dimensions of one row (128 B, coalesced), a ballot per bit-plane yields the packed 32-bit
// word, words are staged in shared memory and leave as 512-byte coalesced 128-bit stores.
constexpr int QP_WARPS = 8;
constexpr int QP_PLANE_STRIDE = 132;  // 32 rows * 4 words + 4 pad words: conflict-free staging

template <typename T>
__global__ void __launch_bounds__(QP_WARPS * 32)
quantize_pack_kernel(const T *__restrict__ x, int64_t n, int dim, int64_t ld, double scale, int width,
                     int C, uint4 *__restrict__ out, unsigned long long *__restrict__ nonfinite) {
    __shared__ __align__(16) uint32_t stage[QP_WARPS][XFBQ_MAX_WIDTH * QP_PLANE_STRIDE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double half = static_cast<double>(1 << (width - 1));
    const int64_t nb = (n + 31) >> 5;
    unsigned long long bad = 0;
    uint32_t *st = stage[warp];
    const int my_plane = lane >> 2, my_t = lane & 3;
    for (int64_t b = static_cast<int64_t>(blockIdx.x) * QP_WARPS + warp; b < nb;
         b += static_cast<int64_t>(gridDim.x) * QP_WARPS) {
        for (int c = 0; c < C; ++c) {
#pragma unroll 2
            for (int r = 0; r < 32; ++r) {
                const int64_t doc = b * 32 + r;
                T v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int k = c * 128 + t * 32 + lane;
                    v[t] = (doc < n && k < dim) ? x[doc * ld + k] : static_cast<T>(0);
                }
                uint32_t mine = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int k = c * 128 + t * 32 + lane;
                    const bool real = (doc < n && k < dim);
                    const unsigned code = real ? quantize_one<T>(v[t], scale, half, bad) : 0u;
#pragma unroll
                    for (int i = 0; i < XFBQ_MAX_WIDTH; ++i) {
                        if (i < width) {  // warp-uniform
                            const uint32_t w = __ballot_sync(0xffffffffu, real && ((code >> i) & 1u));
                            if (lane == i * 4 + t) mine = w;
                        }
                    }
                }
                if (my_plane < width) st[my_plane * QP_PLANE_STRIDE + r * 4 + my_t] = mine;
            }
            __syncwarp();
            for (int i = 0; i < width; ++i) {
                const uint4 w = *reinterpret_cast<const uint4 *>(&st[i * QP_PLANE_STRIDE + lane * 4]);
                out[((b * width + i) * C + c) * 32 + lane] = w;
            }
            __syncwarp();
        }
    }
    if (bad) atomicAdd(nonfinite, bad);
}


// Fast quantizer for float32 rows (16-byte aligned, dim % 4 == 0).  Same result as quantize_one for every
// input, with float64 touched only near a code boundary.  The clip range [-1/scale, 1/scale) is mapped onto the
// whole int32 range, one code = 2^(32-w) integers:
//   Z = cvt.rmi.s32.f32( fma(x, fl32(scale * 2^31), 1024) )        (the conversion saturates: quant.py:147's clip for free)
//   code = top w bits of (Z xor 0x7FFFFFFF)                          (= 2^(w-1) - 1 - (Z >> (32-w)), quant.py:148)
// fl32(scale * 2^31) and the fused multiply-add each carry a relative error <= 2^-24, i.e. together < 257 integers for
// in-range values, so when the low 32-w bits of Z lie in [2048, 2^(32-w)) the exact product lies strictly inside the
// same code step, and so does the float64 value the reference floors (quant.py:146; its own rounding is 2^-22 of an
// integer).  Values beyond the range saturate to the end codes like the reference's clip; the lower end is lifted to
// INT_MIN + 2048 so that it does not look like a boundary.  Everything else -- a value within 2^-21 of the range from a
// code boundary (x = 0 sits exactly on one: its code is right, float multiplication keeps zero exact), about 1 element in
// 10^5 (4-bit) to 10^4 (8-bit) -- is caught by a per-8-elements minimum of the masked low bits and re-examined after the
// branch-free loop; the truly ambiguous ones are redone in float64.  Non-finite inputs poison a running fma(x, 0, acc)
// and take the same route (quant.py:142-143).  Per element: 2 FFMA, F2I, VIMNMX, LOP3, half a VIMNMX3, SHF (codes wider
// than 4 bits: two more shifts).
// A lane owns 32 dimensions of one document (8 LDG.128 in flight; which ones: see the load mapping in the kernel), builds
// their bits of every plane in registers, and the warp's stores of one plane are 128 contiguous bytes of the bundle layout.
// 4x4 bit-block transpose of four 32-bit words (delta swaps; its own inverse): plane words <-> nibble words
__device__ __forceinline__ void transpose_4x4_blocks(uint32_t &p0, uint32_t &p1, uint32_t &p2, uint32_t &p3) {
    uint32_t t;
    t = ((p0 >> 1) ^ p1) & 0x55555555u; p1 ^= t; p0 ^= t << 1;
    t = ((p2 >> 1) ^ p3) & 0x55555555u; p3 ^= t; p2 ^= t << 1;
    t = ((p0 >> 2) ^ p2) & 0x33333333u; p2 ^= t; p0 ^= t << 2;
    t = ((p1 >> 2) ^ p3) & 0x33333333u; p3 ^= t; p1 ^= t << 2;
}

constexpr int QF_WIN = 1024;  // half width of the boundary window, in int32 units of the mapped range

template <int WIDTH>
__device__ __forceinline__ int quant_fast_z(float e, float s32) {
    return max(__float2int_rd(fmaf(e, s32, static_cast<float>(QF_WIN))), INT_MIN + 2 * QF_WIN);
}

template <int WIDTH>
__global__ void __launch_bounds__(256)
quantize_pack_f32_fast_kernel(const float *__restrict__ x, int64_t n, int dim, int64_t ld, double scale,
                              int C, uint32_t *__restrict__ out, unsigned long long *__restrict__ nonfinite) {
    const int lane = threadIdx.x & 31;
    const int d = lane >> 2, t = lane & 3;
    constexpr int SH = 32 - WIDTH;
    constexpr int MASK = static_cast<int>(((1u << SH) - 1u) & ~(2u * QF_WIN - 1u));  // low bits of a step, minus the window
    const double half = static_cast<double>(1 << (WIDTH - 1));
    const float s32 = static_cast<float>(scale * 2147483648.0);
    const int64_t nb = (n + 31) >> 5;
    const int64_t units = nb * C * 4;  // (bundle, chunk, group of 8 documents)
    // Load mapping.  A warp takes 8 documents x 128 dimensions; the four lanes of a document share each 128-byte line:
    // load j = 2 t' + h of lane t fetches dimensions 32 t' + 8 t + 4 h .. + 3, so one load instruction touches 8 lines
    // (one per document), not 32 -- the L1 looks up one line per cycle, and with a lane owning 32 CONSECUTIVE
    // dimensions (32 lines per instruction, 16 bytes each) the kernel sat at 16 B/clk/SM = 4.4 TB/s whatever the ALU
    // work.  A lane's element 4 j + q is then bit 8 t + (4 h + q) of plane word t': byte t' of the lane's plane word
    // belongs to output word t', at byte position t -- a 4 x 4 byte transpose among the four lanes, two rounds of one
    // shuffle and one byte permute per plane, and lane t ends up with output word t.
    const uint32_t sel1 = (t & 1) ? 0x3715u : 0x6240u;  // round 1 (partner t ^ 1): [even source, odd source] x [dest parity of t, + 2]
    const uint32_t sel2 = (t & 2) ? 0x3276u : 0x5410u;  // round 2 (partner t ^ 2): sources 0..3 of this lane's own word
    unsigned long long bad = 0;
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < units;
         u += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const int s8 = static_cast<int>(u & 3);
        const int64_t bc = u >> 2;
        const int c = static_cast<int>(bc % C);
        const int64_t b = bc / C;
        const int64_t doc = b * 32 + s8 * 8 + d;
        const float *src = x + doc * ld + c * 128 + 8 * t;
        // dimensions of this chunk that exist (dim % 4 == 0: whole float4s), none for a padding document
        const int nvc = doc < n ? min(max(dim - c * 128, 0), 128) - 8 * t : 0;
        float4 v[8];
        uint32_t valid = 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int off = 32 * (j >> 1) + 4 * (j & 1);
            const bool ok = off < nvc;
            v[j] = ok ? __ldg(reinterpret_cast<const float4 *>(src + off)) : make_float4(0.f, 0.f, 0.f, 0.f);
            valid |= ok ? 0xFu << (4 * j) : 0u;
        }
        // Codes are collected as nibbles (word q: nibble j = element 4j + q) and turned into bit planes by one 4 x 4
        // bit-block transpose per 32 elements; codes wider than 4 bits as two nibbles (the top 8 bits of Z).
        constexpr bool WIDE = WIDTH > 4;
        uint32_t w[4] = {0u, 0u, 0u, 0u}, wl[4] = {0u, 0u, 0u, 0u};
        int m[4] = {MASK, MASK, MASK, MASK};  // per 8 elements: minimum of the masked low bits (0 = somebody is near a boundary)
        float poison = 0.0f;                  // NaN once any element is not finite
#pragma unroll
        for (int j = 7; j >= 0; --j) {        // nibbles are shifted in from the bottom: last one first
            const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            int z[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                z[q] = quant_fast_z<WIDTH>(e[q], s32);
                poison = fmaf(e[q], 0.0f, poison);
                w[q] = __funnelshift_l(static_cast<uint32_t>(z[q]), w[q], 4);            // bits 31..28 of Z
                if (WIDE) wl[q] = __funnelshift_l(static_cast<uint32_t>(z[q]) << 4, wl[q], 4);  // bits 27..24
            }
            m[j >> 1] = min(min(m[j >> 1], z[0] & MASK), z[1] & MASK);
            m[j >> 1] = min(min(m[j >> 1], z[2] & MASK), z[3] & MASK);
        }
        uint32_t p[WIDTH];  // p[i] = bit plane i of the lane's 32 elements
#pragma unroll
        for (int q = 0; q < 4; ++q) { w[q] ^= 0x77777777u; wl[q] = ~wl[q]; }  // the code is the top WIDTH bits of Z xor 0x7FFFFFFF (quant.py:147-148)
        transpose_4x4_blocks(w[0], w[1], w[2], w[3]);   // -> w[i] = bit 28 + i of every Z
        if (WIDE) transpose_4x4_blocks(wl[0], wl[1], wl[2], wl[3]);   // -> wl[i] = bit 24 + i
#pragma unroll
        for (int i = 0; i < WIDTH; ++i) {   // code bit i = bit 32 - WIDTH + i of Z
            const int zb = 32 - WIDTH + i;
            p[i] = zb >= 28 ? w[zb - 28] : wl[zb >= 24 ? zb - 24 : 0];
        }
        uint32_t groups = 0u;
        const bool poisoned = !(poison == poison);
#pragma unroll
        for (int g = 0; g < 4; ++g) if ((m[g] == 0 || poisoned) && 32 * g < nvc) groups |= 1u << g;
        while (groups) {  // rare: look at the group's elements again; exact float64 path for the ambiguous ones (re-read through L1)
            const int g = __ffs(groups) - 1;
            groups &= groups - 1;
            for (int r = 0; r < 8; ++r) {
                const int pos = 8 * g + r;
                if (!((valid >> pos) & 1u)) break;
                const float e = src[32 * g + r];
                const int z = quant_fast_z<WIDTH>(e, s32);
                if (((z & MASK) == 0 && e != 0.0f) || !(fabsf(e) <= 3.402823466e38f)) {
                    const unsigned code = quantize_one<float>(e, scale, half, bad);
#pragma unroll
                    for (int i = 0; i < WIDTH; ++i) p[i] = (p[i] & ~(1u << pos)) | (((code >> i) & 1u) << pos);
                }
            }
        }
        __syncwarp();
        // bundle layout: 16-byte word ((b * width + i) * C + c) * 32 + doc-in-bundle, 32-bit word t
        const int64_t lane_word = static_cast<int64_t>(s8 * 8 + d) * 4 + t;
#pragma unroll
        for (int i = 0; i < WIDTH; ++i) {
            const uint32_t mine = p[i] & valid;
            const uint32_t x1 = __byte_perm(mine, __shfl_xor_sync(0xffffffffu, mine, 1), sel1);
            const uint32_t x2 = __byte_perm(x1, __shfl_xor_sync(0xffffffffu, x1, 2), sel2);
            out[(((b * WIDTH + i) * C + c) * 32) * 4 + lane_word] = x2;
        }
    }
    if (bad) atomicAdd(nonfinite, bad);
}

// Queries: one warp per query row, output uint32 [nq][width][4C].
template <typename T>
__global__ void __launch_bounds__(256)
quantize_queries_kernel(const T *__restrict__ x, int64_t nq, int dim, int64_t ld, double scale,
                        int width, int C, uint32_t *__restrict__ out,
                        unsigned long long *__restrict__ nonfinite) {
    const int lane = threadIdx.x & 31;
    const int64_t q = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (q >= nq) return;  // whole warp exits together
    const double half = static_cast<double>(1 << (width - 1));
    const int W = 4 * C;
    unsigned long long bad = 0;
    for (int t = 0; t < W; ++t) {
        const int k = t * 32 + lane;
        const bool real = k < dim;
        const unsigned code = real ? quantize_one<T>(x[q * ld + k], scale, half, bad) : 0u;
        for (int i = 0; i < width; ++i) {
            const uint32_t w = __ballot_sync(0xffffffffu, real && ((code >> i) & 1u));
            if (lane == i) out[(q * width + i) * W + t] = w;
        }
    }
    if (bad) atomicAdd(nonfinite, bad);
}

// ----------------------------------------------------------------------------------------------
// Layout conversion: reference planes (width, W64, n) uint64  <->  bundle layout.
// ----------------------------------------------------------------------------------------------
__global__ void planes_to_bundles_kernel(const uint64_t *__restrict__ planes, int64_t n, int W64,
                                         int width, int C, uint4 *__restrict__ out, int64_t total) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int lane = static_cast<int>(e & 31);
    int64_t r = e >> 5;
    const int c = static_cast<int>(r % C); r /= C;
    const int i = static_cast<int>(r % width);
    const int64_t b = r / width;
    const int64_t doc = b * 32 + lane;
    uint64_t w0 = 0, w1 = 0;
    if (doc < n) {
        if (2 * c < W64) w0 = planes[(static_cast<int64_t>(i) * W64 + 2 * c) * n + doc];
        if (2 * c + 1 < W64) w1 = planes[(static_cast<int64_t>(i) * W64 + 2 * c + 1) * n + doc];
    }
    out[e] = make_uint4(static_cast<uint32_t>(w0), static_cast<uint32_t>(w0 >> 32),
                        static_cast<uint32_t>(w1), static_cast<uint32_t>(w1 >> 32));
}

__global__ void bundles_to_planes_kernel(const uint4 *__restrict__ db, int64_t n, int W64, int width,
                                         int C, uint64_t *__restrict__ planes, int64_t total) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int lane = static_cast<int>(e & 31);
    int64_t r = e >> 5;
    const int c = static_cast<int>(r % C); r /= C;
    const int i = static_cast<int>(r % width);
    const int64_t b = r / width;
    const int64_t doc = b * 32 + lane;
    if (doc >= n) return;
    const uint4 w = db[e];
    if (2 * c < W64)
        planes[(static_cast<int64_t>(i) * W64 + 2 * c) * n + doc] = static_cast<uint64_t>(w.x) | (static_cast<uint64_t>(w.y) << 32);
    if (2 * c + 1 < W64)
        planes[(static_cast<int64_t>(i) * W64 + 2 * c + 1) * n + doc] = static_cast<uint64_t>(w.z) | (static_cast<uint64_t>(w.w) << 32);
}

// ----------------------------------------------------------------------------------------------
// Distance arithmetic (_kernels.py:56-69):
//   d = sum_{i<wd} sum_{j<wq} sum_w popcount(D[i,w] ^ Q[j,w]) << (i+j)
// grouped by weight class s = i+j so each class is shifted once.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t popc4(const uint4 a, const uint4 b) {
    return __popc(a.x ^ b.x) + __popc(a.y ^ b.y) + __popc(a.z ^ b.z) + __popc(a.w ^ b.w);
}

// Generic widths / dims: document words are re-read from global (L1/L2) for every query.
__device__ __forceinline__ uint32_t distance_generic(const uint4 *__restrict__ doc /* + lane */, int wd, int C,
                                                     const uint32_t *qs, int wq) {
    uint32_t d = 0;
    for (int i = 0; i < wd; ++i)
        for (int c = 0; c < C; ++c) {
            const uint4 x = __ldg(doc + (i * C + c) * 32);
            for (int j = 0; j < wq; ++j) {
                const uint4 y = *reinterpret_cast<const uint4 *>(qs + (j * C + c) * 4);
                d += popc4(x, y) << (i + j);
            }
        }
    return d;
}

template <int WD, int WQ, int C>
__device__ __forceinline__ uint32_t distance_regs(const uint4 (&x)[WD * C], const uint32_t *qs) {
    uint32_t acc[WD + WQ - 1];
#pragma unroll
    for (int s = 0; s < WD + WQ - 1; ++s) acc[s] = 0;
#pragma unroll
    for (int j = 0; j < WQ; ++j)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const uint4 y = *reinterpret_cast<const uint4 *>(qs + (j * C + c) * 4);  // broadcast LDS.128
#pragma unroll
            for (int i = 0; i < WD; ++i) acc[i + j] += popc4(x[i * C + c], y);
        }
    uint32_t d = 0;
#pragma unroll
    for (int s = 0; s < WD + WQ - 1; ++s) d += acc[s] << s;
    return d;
}

__global__ void __launch_bounds__(256)
batch_distances_kernel(const uint4 *__restrict__ db, int64_t n, int wd, int C,
                       const uint32_t *__restrict__ q, int wq, uint64_t *__restrict__ out) {
    extern __shared__ __align__(16) uint32_t qs_dyn[];
    const int qwords = wq * C * 4;
    for (int t = threadIdx.x; t < qwords; t += blockDim.x) qs_dyn[t] = q[t];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nb = (n + 31) >> 5;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        const int64_t doc = b * 32 + lane;
        const uint32_t d = distance_generic(db + b * wd * C * 32 + lane, wd, C, qs_dyn, wq);
        if (doc < n) out[doc] = d;
    }
}

// Candidate gather of k_select (search.py:206-216: histogram threshold, then every row with d <= threshold):
// one pass over the codes, no distance array.  counts[0] += rows with d <= threshold; the first `cap` of them
// (in no particular order) go to ids_out.
__global__ void __launch_bounds__(256)
collect_candidates_kernel(const uint4 *__restrict__ db, int64_t n, int wd, int C, const uint32_t *__restrict__ q, int wq,
                          uint32_t threshold, int64_t *__restrict__ ids_out, int64_t cap, unsigned long long *__restrict__ counts) {
    extern __shared__ __align__(16) uint32_t qs_dyn[];
    const int qwords = wq * C * 4;
    for (int t = threadIdx.x; t < qwords; t += blockDim.x) qs_dyn[t] = q[t];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nb = (n + 31) >> 5;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        const int64_t doc = b * 32 + lane;
        const uint32_t d = distance_generic(db + b * wd * C * 32 + lane, wd, C, qs_dyn, wq);
        const bool hit = doc < n && d <= threshold;
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

// Same, for the common widths: the document's words are loaded first (WD * C independent LDG.128), the
// weight classes accumulate in registers.
template <int WD, int WQ, int C>
__global__ void __launch_bounds__(256)
collect_candidates_fast_kernel(const uint4 *__restrict__ db, int64_t n, const uint32_t *__restrict__ q, uint32_t threshold,
                               int64_t *__restrict__ ids_out, int64_t cap, unsigned long long *__restrict__ counts) {
    __shared__ __align__(16) uint32_t qs[WQ * C * 4];
    for (int t = threadIdx.x; t < WQ * C * 4; t += blockDim.x) qs[t] = q[t];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nb = (n + 31) >> 5;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        const int64_t doc = b * 32 + lane;
        uint4 x[WD * C];
#pragma unroll
        for (int e = 0; e < WD * C; ++e) x[e] = __ldg(db + (b * (WD * C) + e) * 32 + lane);
        const uint32_t d = distance_regs<WD, WQ, C>(x, qs);
        const bool hit = doc < n && d <= threshold;
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

// ----------------------------------------------------------------------------------------------
// Top-K selection state of one CTA: per query slot a candidate list in shared memory, a count
// and a threshold key.  A score enters the list only if its key (distance<<32 | row id) is below
// the threshold; when a list cannot take another full step (SCAN_THREADS pushes) it is sorted,
// cut to the k best and the threshold becomes the k-th key (search.py:129-131 order).
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ void bitonic_sort_block(uint64_t *s, int P) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = s[lo], b = s[hi];
                if ((a > b) == up) { s[lo] = b; s[hi] = a; }
            }
            __syncthreads();
        }
}

__device__ __forceinline__ int pow2_ceil(int v) {
    int p = 2;
    while (p < v) p <<= 1;
    return p;
}

// Block-wide; every thread must call it with the same arguments.
__device__ void compact_list(uint64_t *list, uint32_t *cnt_p, uint64_t *thr_p, int k) {
    const int c = static_cast<int>(*cnt_p);
    const int P = pow2_ceil(c);
    __syncthreads();  // everyone has read *cnt_p
    for (int t = c + threadIdx.x; t < P; t += blockDim.x) list[t] = KEY_INF;
    __syncthreads();
    bitonic_sort_block(list, P);
    if (threadIdx.x == 0) {
        *cnt_p = static_cast<uint32_t>(c < k ? c : k);
        *thr_p = (c >= k) ? list[k - 1] : KEY_INF;
    }
    __syncthreads();
}

__device__ __forceinline__ void push_candidate(bool pass, uint64_t key, uint64_t *list, uint32_t *cnt_p, int lane) {
    const unsigned m = __ballot_sync(0xffffffffu, pass);
    if (m == 0) return;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cnt_p, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pass) list[base + __popc(m & ((1u << lane) - 1u))] = key;
}

struct ScanParams {
    const uint4 *db;
    int64_t n;
    int64_t row_offset;
    const uint32_t *q;
    uint64_t *out;        // [splits][nq][k]
    int64_t nq;
    int64_t split_steps;  // steps (of SCAN_WARPS bundles) per doc split
    int wd, wq, C;
    int k, cap, tq;
};

inline size_t scan_smem_bytes(int tq, int qwords, int cap) {
    // cand + thr (8B) ; qs must stay 16-byte aligned -> pad thr to even count
    const size_t thr_slots = (tq + 1) & ~1;
    return static_cast<size_t>(tq) * cap * 8 + thr_slots * 8 + static_cast<size_t>(tq) * qwords * 4 + static_cast<size_t>(tq) * 4 + 16;
}

// WD == 0 selects the generic (runtime widths) body.
template <int WD, int WQ, int CC>
__global__ void __launch_bounds__(SCAN_THREADS, (WD == 0 ? 1 : 2))
scan_topk_kernel(const ScanParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int wd = WD ? WD : p.wd, wq = WD ? WQ : p.wq, C = WD ? CC : p.C;
    const int qwords = wq * C * 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q0 = static_cast<int64_t>(blockIdx.y) * p.tq;
    const int tq = static_cast<int>(min(static_cast<int64_t>(p.tq), p.nq - q0));
    const int thr_slots = (p.tq + 1) & ~1;
    // carve with the launch-time tq so offsets match scan_smem_bytes
    uint64_t *cand = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *thr = cand + static_cast<size_t>(p.tq) * p.cap;
    uint32_t *qs = reinterpret_cast<uint32_t *>(thr + thr_slots);
    uint32_t *cnt = qs + static_cast<size_t>(p.tq) * qwords;

    for (int t = threadIdx.x; t < tq * qwords; t += SCAN_THREADS) qs[t] = p.q[q0 * qwords + t];
    for (int t = threadIdx.x; t < tq; t += SCAN_THREADS) { thr[t] = KEY_INF; cnt[t] = 0; }
    __syncthreads();

    const int64_t nb = (p.n + 31) >> 5;
    const int64_t step0 = static_cast<int64_t>(blockIdx.x) * p.split_steps;
    int64_t b_begin = step0 * SCAN_WARPS;
    int64_t b_end = min(nb, (step0 + p.split_steps) * SCAN_WARPS);
    const int64_t bundle_words = static_cast<int64_t>(wd) * C * 32;  // uint4 per bundle

    uint4 cur[WD ? WD * CC : 1];
    uint4 nxt[WD ? WD * CC : 1];
    if (WD) {
        const int64_t b = b_begin + warp;
        if (b < b_end) {
#pragma unroll
            for (int e = 0; e < (WD ? WD * CC : 1); ++e) cur[e] = __ldg(p.db + b * bundle_words + e * 32 + lane);
        }
    }

    for (int64_t bs = b_begin; bs < b_end; bs += SCAN_WARPS) {
        const int64_t b = bs + warp;
        const bool active = b < b_end;
        if (WD) {
            const int64_t bn = b + SCAN_WARPS;
            if (bn < b_end) {
#pragma unroll
                for (int e = 0; e < (WD ? WD * CC : 1); ++e) nxt[e] = __ldg(p.db + bn * bundle_words + e * 32 + lane);
            }
        }
        if (active) {  // warp-uniform
            const int64_t doc = b * 32 + lane;
            const bool valid = doc < p.n;
            const uint64_t gid = static_cast<uint64_t>(p.row_offset + doc);
            const uint4 *dptr = p.db + b * bundle_words + lane;
            for (int qi = 0; qi < tq; ++qi) {
                uint32_t d;
                if (WD) d = distance_regs<(WD ? WD : 1), (WD ? WQ : 1), (WD ? CC : 1)>(cur, qs + qi * qwords);
                else d = distance_generic(dptr, wd, C, qs + qi * qwords, wq);
                const uint64_t key = (static_cast<uint64_t>(d) << 32) | gid;
                const bool pass = valid && key < thr[qi];
                push_candidate(pass, key, cand + static_cast<size_t>(qi) * p.cap, cnt + qi, lane);
            }
        }
        if (WD) {
#pragma unroll
            for (int e = 0; e < (WD ? WD * CC : 1); ++e) cur[e] = nxt[e];
        }
        bool need = false;
        __syncthreads();
        for (int qi = threadIdx.x; qi < tq; qi += SCAN_THREADS) need |= cnt[qi] > static_cast<uint32_t>(p.cap - SCAN_THREADS);
        if (__syncthreads_or(need)) {
            for (int qi = 0; qi < tq; ++qi)
                if (cnt[qi] > static_cast<uint32_t>(p.cap - SCAN_THREADS))
                    compact_list(cand + static_cast<size_t>(qi) * p.cap, cnt + qi, thr + qi, p.k);
        }
    }
    __syncthreads();
    for (int qi = 0; qi < tq; ++qi) {
        uint64_t *list = cand + static_cast<size_t>(qi) * p.cap;
        compact_list(list, cnt + qi, thr + qi, p.k);
        const int c = static_cast<int>(cnt[qi]);
        uint64_t *dst = p.out + (static_cast<int64_t>(blockIdx.x) * p.nq + q0 + qi) * p.k;
        for (int t = threadIdx.x; t < p.k; t += SCAN_THREADS) dst[t] = t < c ? list[t] : KEY_INF;
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------------------------
// Merge: one CTA per query keeps the K2 = pow2 >= k best keys in the lower half of a 2*K2
// buffer, streams the parts through the upper half and re-sorts.
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
merge_topk_kernel(const uint64_t *__restrict__ in, int parts, int64_t nq, int k, int K2,
                  uint64_t *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *buf = reinterpret_cast<uint64_t *>(smem_raw);
    const int64_t q = blockIdx.x;
    for (int t = threadIdx.x; t < K2; t += blockDim.x) buf[t] = KEY_INF;
    const int64_t total = static_cast<int64_t>(parts) * k;
    for (int64_t base = 0; base < total; base += K2) {
        for (int t = threadIdx.x; t < K2; t += blockDim.x) {
            const int64_t e = base + t;
            uint64_t v = KEY_INF;
            if (e < total) {
                const int64_t part = e / k, slot = e % k;
                v = in[(part * nq + q) * k + slot];
            }
            buf[K2 + t] = v;
        }
        __syncthreads();
        bitonic_sort_block(buf, 2 * K2);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < k; t += blockDim.x) out[q * k + t] = buf[t];
}

// Tree merge: one CTA per (group of up to G parts, query).  Every part row is sorted, so two
// rows A, B of length K2 reduce to the K2 smallest of their union by c_i = min(A_i, B_{K2-1-i})
// (a bitonic sequence) followed by log2(K2) bitonic-merge stages; log2(G) rounds leave the answer
// in row 0.  Far fewer barrier stages than re-sorting, so single-query latency stays small.
template <int K2, bool SORT>
__global__ void __launch_bounds__(512)
merge_tree_kernel(const uint64_t *__restrict__ in, int parts, int64_t nq, int k, int G,
                  uint64_t *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *buf = reinterpret_cast<uint64_t *>(smem_raw);
    const int64_t q = blockIdx.y;
    const int p0 = blockIdx.x * G;
    const int rows = min(G, parts - p0);
    int active = 1;
    while (active < rows) active <<= 1;
    for (int idx = threadIdx.x; idx < active * K2; idx += blockDim.x) {
        const int r = idx / K2, i = idx % K2;
        buf[idx] = (r < rows && i < k) ? in[((static_cast<int64_t>(p0) + r) * nq + q) * k + i] : KEY_INF;
    }
    __syncthreads();
    if (SORT) {  // rows arrive unsorted (tensor engine emits its lists as they are): bitonic sort of every row
        for (int size = 2; size <= K2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int idx = threadIdx.x; idx < active * (K2 >> 1); idx += blockDim.x) {
                    const int r = idx / (K2 >> 1), t = idx % (K2 >> 1);
                    const int c = 2 * t - (t & (stride - 1));
                    const int lo = r * K2 + c, hi = lo + stride;
                    const bool up = (c & size) == 0;
                    const uint64_t a = buf[lo], b = buf[hi];
                    if ((a > b) == up) { buf[lo] = b; buf[hi] = a; }
                }
                __syncthreads();
            }
    }
    while (active > 1) {
        const int half = active >> 1;
        for (int idx = threadIdx.x; idx < half * K2; idx += blockDim.x) {
            const int r = idx / K2, i = idx % K2;
            const uint64_t a = buf[r * K2 + i], b = buf[(r + half) * K2 + (K2 - 1 - i)];
            buf[r * K2 + i] = a < b ? a : b;
        }
        __syncthreads();
#pragma unroll 1
        for (int stride = K2 >> 1; stride > 0; stride >>= 1) {
            for (int idx = threadIdx.x; idx < half * (K2 >> 1); idx += blockDim.x) {
                const int r = idx / (K2 >> 1), t = idx % (K2 >> 1);
                const int lo = r * K2 + 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const uint64_t a = buf[lo], b = buf[hi];
                if (a > b) { buf[lo] = b; buf[hi] = a; }
            }
            __syncthreads();
        }
        active = half;
    }
    uint64_t *dst = out + (static_cast<int64_t>(blockIdx.x) * nq + q) * k;
    for (int i = threadIdx.x; i < k; i += blockDim.x) dst[i] = buf[i];
}


// Bounded merge (tensor engine, seeded scans): bound[q] is a proven lower bound of query q's k-th best score
// (the shared threshold the scan CTAs tightened), so a partial-result key with a larger distance than
// Dq - bound cannot be in the answer.  One CTA per query drops those keys while loading -- typically little
// more than k of the parts * k survive -- and sorts only the survivors (next power of two), instead of sorting
// and tree-merging every row (config 4: 0.47 ms -> 0.05 ms).  Rows may arrive unsorted.  Exact for any number of
// survivors: when the buffer of B keys could overflow it is sorted, cut back to its k best, and the bound
// tightens to the k-th of those.  B is a power of two >= k + blockDim.x.  With bound == nullptr the rows must be
// sorted and the bound comes from the rows themselves (see below).
// Block-wide bounded merge: keeps, of `total` keys delivered by fetch(e) (KEY_INF = no key), those with distance <= limit in a
// shared-memory buffer of B keys (a power of two >= k + blockDim.x), sorts the survivors and writes the k best to dst
// (KEY_INF padded).  Exact for any number of survivors: when the buffer could overflow it is sorted, cut back to its k best,
// and the limit tightens to the k-th of those.  Every thread of the block calls it with the same arguments.
template <class Fetch>
__device__ void merge_bounded_block(uint64_t *buf, int B, int k, int64_t total, long long limit0, Fetch fetch, uint64_t *dst) {
    __shared__ int s_cnt;
    __shared__ long long s_limit;
    const int lane = threadIdx.x & 31, nt = blockDim.x;
    if (threadIdx.x == 0) { s_cnt = 0; s_limit = limit0; }
    auto sort_prefix = [&](int c) {  // ascending sort of buf[0, c), padded to a power of two; ends on a barrier
        int n2 = 32;
        while (n2 < c) n2 <<= 1;
        for (int i = c + threadIdx.x; i < n2; i += nt) buf[i] = KEY_INF;
        __syncthreads();
        for (int size = 2; size <= n2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < (n2 >> 1); t += nt) {
                    const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const uint64_t a = buf[lo], b = buf[hi];
                    if ((a > b) == up) { buf[lo] = b; buf[hi] = a; }
                }
                __syncthreads();
            }
    };
    for (int64_t e0 = 0; e0 < total; e0 += nt) {
        __syncthreads();
        const int c = s_cnt;
        __syncthreads();  // every thread has read the count before any warp appends: the branch below is block-uniform
        if (c + nt > B) {  // the next round of appends could overflow: keep the k best, tighten the bound
            sort_prefix(c);
            if (threadIdx.x == 0) {
                s_cnt = c < k ? c : k;
                if (c >= k) {
                    const long long kth = static_cast<long long>(buf[k - 1] >> 32);
                    if (kth < s_limit) s_limit = kth;
                }
            }
            __syncthreads();
        }
        const long long limit = s_limit;
        const int64_t e = e0 + threadIdx.x;
        const uint64_t key = e < total ? fetch(e) : KEY_INF;
        const bool keep = key != KEY_INF && static_cast<long long>(key >> 32) <= limit;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(&s_cnt, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) buf[base + __popc(m & ((1u << lane) - 1u))] = key;
    }
    __syncthreads();
    const int c = s_cnt;
    sort_prefix(c);
    for (int i = threadIdx.x; i < k; i += nt) dst[i] = i < c ? buf[i] : KEY_INF;
}

// Block-wide: s_pre[i] = sum of len(j) for j < i, i = 0 .. parts (lists of different lengths, flat entry index ->
// (list, slot) by binary search).  The lengths are fetched by all threads at once (one L2 round trip instead of one per 32
// lists), then warp 0 scans them in shared memory.  Ends without a barrier: the caller synchronises.
template <class Len>
__device__ void prefix_lengths(int *s_pre, int parts, Len len) {
    for (int part = threadIdx.x; part < parts; part += blockDim.x) s_pre[part] = len(part);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int run = 0;
        for (int p0 = 0; p0 < parts; p0 += 32) {
            const int part = p0 + lane;
            const int c = part < parts ? s_pre[part] : 0;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            if (part < parts) s_pre[part] = run + inc - c;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_pre[parts] = run;
    }
}
__device__ __forceinline__ int find_part(const int *s_pre, int parts, int e) {  // largest part with s_pre[part] <= e
    int lo = 0, hi = parts;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pre[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

// With `src.counts` the partial results are the scan CTAs' candidate lists where they lie (single-wave plans of the queue
// kernel: CTA part * groups + group holds, for each of its nq_cta queries, src.counts[...] <= cap unsorted keys): the rows
// have different lengths, entry e of the query maps to (part, slot) through a prefix sum of the lengths.
struct ListSrc {
    const int *counts = nullptr;  // [parts * groups][nq_cta]
    int nq_cta = 0, cap = 0, groups = 0;
};
__global__ void __launch_bounds__(512)
merge_bounded_kernel(const uint64_t *__restrict__ in, int parts, int64_t nq, int k, int B, const int32_t *__restrict__ bound,
                     const int32_t *__restrict__ qconst, uint64_t *__restrict__ out, const ListSrc src = ListSrc()) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *buf = reinterpret_cast<uint64_t *>(smem_raw);
    __shared__ long long s_rows_limit;
    __shared__ int s_pre[257];  // list mode: entries of the query in parts < i (parts <= 256)
    const int64_t q = blockIdx.x;
    const int nt = blockDim.x;
    const bool lists = src.counts != nullptr;
    const int gr = lists ? static_cast<int>(q / src.nq_cta) : 0, ql = lists ? static_cast<int>(q - static_cast<int64_t>(gr) * src.nq_cta) : 0;
    if (lists) {
        prefix_lengths(s_pre, parts, [&](int part) { return src.counts[(static_cast<int64_t>(part) * src.groups + gr) * src.nq_cta + ql]; });
        __syncthreads();
    }
    // largest distance that can still be in the top k
    long long limit = bound ? static_cast<long long>(qconst[q]) - static_cast<long long>(bound[q]) : -1;
    if (!bound) {
        // Sorted rows without a shared threshold (last level of a tree merge): the m-th keys of all rows, m = ceil(k / parts),
        // bound the answer -- parts * m >= k keys are no larger than the largest of them.
        if (threadIdx.x == 0) s_rows_limit = -1;
        __syncthreads();
        const int m = (k + parts - 1) / parts;
        long long mine = -1;
        for (int part = threadIdx.x; part < parts; part += nt) {
            const uint64_t key = in[(static_cast<int64_t>(part) * nq + q) * k + (m - 1)];
            const long long d = key == KEY_INF ? 0x7FFFFFFFFFFFFFFFll : static_cast<long long>(key >> 32);
            mine = d > mine ? d : mine;
        }
        atomicMax(&s_rows_limit, mine);
        __syncthreads();
        limit = s_rows_limit;
    }
    const int64_t total = lists ? s_pre[parts] : static_cast<int64_t>(parts) * k;
    merge_bounded_block(buf, B, k, total, limit, [&](int64_t e) -> uint64_t {
        if (lists) {
            const int part = find_part(s_pre, parts, static_cast<int>(e));
            return __ldcg(in + ((static_cast<int64_t>(part) * src.groups + gr) * src.nq_cta + ql) * src.cap + (e - s_pre[part]));
        }
        const int64_t part = e / k, slot = e - part * k;
        return in[(part * nq + q) * k + slot];
    }, out + q * k);
}

}  // namespace
#include "xfbq_mma.cuh"
#include "xfbq_umma.cuh"
#include "xfbq_select.cuh"
#include "xfbq_coop.cuh"
namespace {

__global__ void unpack_keys_kernel(const uint64_t *__restrict__ keys, int64_t count,
                                   int64_t *__restrict__ dist, int64_t *__restrict__ ids) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint64_t key = keys[e];
    if (key == KEY_INF) { dist[e] = -1; ids[e] = -1; }
    else { dist[e] = static_cast<int64_t>(key >> 32); ids[e] = static_cast<int64_t>(key & 0xFFFFFFFFull); }
}

// ----------------------------------------------------------------------------------------------
// Host-side planning shared by xfbq_scan_workspace_bytes and xfbq_scan_topk.
// ----------------------------------------------------------------------------------------------
struct ScanPlan {
    int tq = 1, cap = 0, splits = 1, q_tiles = 1;
    int64_t split_steps = 1;
    size_t smem = 0;
    bool fast = false;
};

typedef void (*ScanKernel)(const ScanParams);

ScanKernel pick_kernel(int wd, int wq, int C) {
#define XFBQ_CASE(WD_, WQ_, C_) if (wd == WD_ && wq == WQ_ && C == C_) return scan_topk_kernel<WD_, WQ_, C_>;
    XFBQ_CASE(3, 4, 1) XFBQ_CASE(3, 4, 2) XFBQ_CASE(3, 4, 4)
    XFBQ_CASE(4, 4, 1) XFBQ_CASE(4, 4, 2) XFBQ_CASE(4, 4, 4)
#undef XFBQ_CASE
    return nullptr;
}

// Plan overrides come from XFBQ_* environment variables.  They are read ONCE, at the first planning call
// of the process, into a snapshot: no getenv on the call path (it is not safe against a concurrent setenv) and a plan cannot
// change between xfbq_scan_workspace_bytes and xfbq_scan_topk.  XFBQ_ENV_LIVE=1 (set before the first call: the test-suite,
// the experiment tools) re-reads the environment on every call instead, so tests can switch plans in-process.
struct EnvSnapshot {
    bool live = false;
    std::unordered_map<std::string, std::string> kv;
};
const EnvSnapshot &env_snapshot() {
    static EnvSnapshot snap;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *live = getenv("XFBQ_ENV_LIVE");
        snap.live = live && *live && strcmp(live, "0") != 0;
        for (char **e = environ; e && *e; ++e) {
            if (strncmp(*e, "XFBQ_", 5) != 0) continue;
            const char *eq = strchr(*e, '=');
            if (eq) snap.kv.emplace(std::string(*e, eq - *e), std::string(eq + 1));
        }
    });
    return snap;
}
const char *env_get(const char *name) {
    const EnvSnapshot &snap = env_snapshot();
    if (snap.live) return getenv(name);
    auto it = snap.kv.find(name);
    return it == snap.kv.end() ? nullptr : it->second.c_str();
}
int env_int(const char *name, int dflt) {
    const char *v = env_get(name);
    if (!v || !*v) return dflt;
    return atoi(v);
}

int make_plan(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k, ScanPlan *plan) {
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    const int C = static_cast<int>(chunks128(dim));
    const int qwords = wq * C * 4;
    ScanPlan pl;
    int cap = 2;
    while (cap < k + SCAN_THREADS) cap <<= 1;
    pl.cap = cap;
    pl.fast = pick_kernel(wd, wq, C) != nullptr && env_int("XFBQ_FORCE_GENERIC", 0) == 0;
    const size_t budget = static_cast<size_t>(info.smem_optin) - 1024;
    int tq_max = env_int("XFBQ_TQ", 32);
    if (tq_max < 1) tq_max = 1;
    int tq = static_cast<int>(nq < tq_max ? nq : tq_max);
    while (tq > 1 && scan_smem_bytes(tq, qwords, cap) > budget) --tq;
    if (scan_smem_bytes(tq, qwords, cap) > budget)
        return fail(XFBQ_E_UNSUPPORTED, "scan needs %zu bytes of shared memory for dim=%lld k=%d, device offers %zu",
                    scan_smem_bytes(tq, qwords, cap), static_cast<long long>(dim), k, budget);
    pl.tq = tq;
    pl.smem = scan_smem_bytes(tq, qwords, cap);
    pl.q_tiles = static_cast<int>((nq + tq - 1) / tq);
    const int64_t steps = (bundles_of(n) + SCAN_WARPS - 1) / SCAN_WARPS;
    // resident CTAs per SM: limited by shared memory (and 2 by launch bounds for the fast kernels)
    int occ = static_cast<int>((static_cast<size_t>(info.smem_optin) + 1024) / (pl.smem + 1024));
    const int occ_cap = pl.fast ? 2 : 1;
    if (occ > occ_cap) occ = occ_cap;
    if (occ < 1) occ = 1;
    const int64_t capacity = static_cast<int64_t>(info.sms) * occ;
    const int64_t want = pl.q_tiles >= capacity ? 4 * capacity : capacity;
    int64_t splits = (want + pl.q_tiles - 1) / pl.q_tiles;
    const int forced = env_int("XFBQ_SPLITS", 0);
    if (forced > 0) splits = forced;
    if (splits > steps) splits = steps;
    if (splits < 1) splits = 1;
    pl.split_steps = (steps + splits - 1) / splits;
    if (pl.split_steps < 1) pl.split_steps = 1;
    pl.splits = static_cast<int>((steps + pl.split_steps - 1) / pl.split_steps);
    if (pl.splits < 1) pl.splits = 1;
    *plan = pl;
    return XFBQ_OK;
}

int merge_k2(int k) {
    int K2 = 32;
    while (K2 < k) K2 <<= 1;
    return K2;
}

// Parts one tree-merge CTA can hold in shared memory (power of two), 0 if K2 is too large.
int merge_group_max(int k) {
    const int K2 = merge_k2(k);
    int G = (160 * 1024) / (K2 * 8);
    if (G < 2) return 0;
    int p = 2;
    while (p * 2 <= G && p * 2 <= 256) p <<= 1;
    return p;
}

int launch_merge_stream(const uint64_t *in, int parts, int64_t nq, int k, uint64_t *out, cudaStream_t st) {
    const int K2 = merge_k2(k);
    const size_t smem = static_cast<size_t>(2) * K2 * 8;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(merge_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "merge smem opt-in: %s", cudaGetErrorString(e));
    }
    merge_topk_kernel<<<static_cast<unsigned>(nq), 256, smem, st>>>(in, parts, nq, k, K2, out);
    return check_launch("merge_topk_kernel");
}

// Level plan of the tree merge: parts per CTA (G) and resulting groups per level.  Small query
// counts use small groups so the first level still spreads over the whole chip.
struct MergeLevels {
    int levels = 0;
    int G[8], groups[8];
    int64_t scratch_parts = 0;  // sum of groups over the non-final levels
};

MergeLevels merge_levels(int parts, int k, int64_t nq) {
    MergeLevels ml;
    const int gmax = merge_group_max(k);
    if (gmax == 0 || parts <= 1) return ml;
    (void)nq;
    while (parts > 1 && ml.levels < 8) {
        // the level before the last one uses the smallest groups that still let the last level
        // finish in one CTA per query, so that it spreads over many SMs
        int G = gmax;
        if (parts > gmax && parts <= gmax * gmax) {
            G = 4;
            while ((parts + G - 1) / G > gmax) G <<= 1;
        }
        const int groups = (parts + G - 1) / G;
        ml.G[ml.levels] = G; ml.groups[ml.levels] = groups;
        if (groups > 1) ml.scratch_parts += groups;
        ++ml.levels;
        parts = groups;
    }
    return ml;
}

int64_t merge_scratch_parts(int parts, int k, int64_t nq) { return merge_levels(parts, k, nq).scratch_parts; }

typedef void (*MergeKernel)(const uint64_t *, int, int64_t, int, int, uint64_t *);

MergeKernel pick_merge_kernel(int K2, bool sort) {
#define XFBQ_MERGE_CASE(K_) case K_: return sort ? merge_tree_kernel<K_, true> : merge_tree_kernel<K_, false>;
    switch (K2) {
        XFBQ_MERGE_CASE(32) XFBQ_MERGE_CASE(64) XFBQ_MERGE_CASE(128) XFBQ_MERGE_CASE(256)
        XFBQ_MERGE_CASE(512) XFBQ_MERGE_CASE(1024) XFBQ_MERGE_CASE(2048) XFBQ_MERGE_CASE(4096)
    }
#undef XFBQ_MERGE_CASE
    return nullptr;
}

int launch_merge(const uint64_t *in, int parts, int64_t nq, int k, uint64_t *out, uint64_t *scratch,
                 cudaStream_t st, bool sort_input = false) {
    MergeLevels ml = merge_levels(parts, k, nq);
    if (sort_input && parts == 1 && merge_group_max(k) > 0) {  // nothing to merge, but the row must be sorted
        ml.levels = 1; ml.G[0] = 1; ml.groups[0] = 1; ml.scratch_parts = 0;
    }
    const bool tree_ok = nq <= 65535 && ml.levels > 0 && !(ml.scratch_parts > 0 && !scratch) && ml.groups[ml.levels - 1] == 1;
    if (!tree_ok) {
        if (sort_input) return fail(XFBQ_E_UNSUPPORTED, "unsorted partial results need the tree merge (parts=%d nq=%lld k=%d)", parts, (long long)nq, k);
        return launch_merge_stream(in, parts, nq, k, out, st);
    }
    const int K2 = merge_k2(k);
    for (int l = 0; l < ml.levels; ++l) {
        MergeKernel kern = pick_merge_kernel(K2, sort_input && l == 0);
        const int G = ml.G[l], groups = ml.groups[l];
        int rows = parts < G ? parts : G, active = 1;
        while (active < rows) active <<= 1;
        const size_t smem = static_cast<size_t>(active) * K2 * 8;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
            if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "merge smem opt-in: %s", cudaGetErrorString(e));
        }
        uint64_t *dst = groups == 1 ? out : scratch;
        if (groups == 1 && rows >= 16 && !(sort_input && l == 0) && k <= 1024 && env_int("XFBQ_MERGE_BOUNDED", 1)) {
            // last level over many sorted rows (single queries: 74 rows of 100): keep what the rows' own m-th keys allow
            // and sort those few hundred keys, instead of log2(rows) rounds of bitonic merges in one CTA (28.6 -> see profiles)
            merge_bounded_kernel<<<static_cast<unsigned>(nq), 512, 4096 * 8, st>>>(in, parts, nq, k, 4096, nullptr, nullptr, out);
            return check_launch("merge_bounded_kernel");
        }
        int threads = active * K2 / 4;
        threads = threads < 64 ? 64 : (threads > 512 ? 512 : threads);
        kern<<<dim3(static_cast<unsigned>(groups), static_cast<unsigned>(nq)), threads, smem, st>>>(in, parts, nq, k, G, dst);
        if (int rc = check_launch("merge_tree_kernel")) return rc;
        if (groups == 1) return XFBQ_OK;
        in = dst;
        scratch += static_cast<int64_t>(groups) * nq * k;
        parts = groups;
    }
    return XFBQ_OK;
}

// Byte-tile geometry of a dimension: CP chunks of 128 dims in the bit planes, CT >= CP chunks per tile (dims above 512 are
// padded to an even chunk count and streamed as KP = 2 K parts of Cp chunks that accumulate into one accumulator).
struct TileGeom { int CP, CT, KP, Cp; };
inline TileGeom tile_geom(int64_t dim) {
    TileGeom g;
    g.CP = static_cast<int>(chunks128(dim));
    g.KP = g.CP > 4 ? 2 : 1;
    g.CT = g.KP == 2 ? (g.CP + 1) & ~1 : g.CP;
    g.Cp = g.CT / g.KP;
    return g;
}

// ----------------------------------------------------------------------------------------------
// Integer-MMA engine planning (kernels in xfbq_mma.cuh).
// ----------------------------------------------------------------------------------------------
struct MmaShape {  // launch geometry of one mma::scan_kernel launch over n documents
    int MT = 2, NT = 2, QPW = 32, QW = 8, DW = 1, groups = 1, grid = 1, slots = 1, parts = 1, cap = 0;
    int RR = 0, BR = 0;  // ring depths (RR = 0: does not fit in shared memory)
    bool fused = false;  // one query warp: tiles go raw ring -> registers -> IMMA, no byte ring
    int warps = mma::WARPS;
    int64_t stages = 0, nq_pad = 0, n_pad = 0;
    size_t smem = 0, lists_bytes = 0, parts_bytes = 0, mscratch_bytes = 0;
};

struct MmaPlan {
    bool ok = false;
    MmaShape main, pre;      // pre: sample scan that seeds the thresholds (small batches only)
    int64_t sample = 0;      // documents in the sample scan, 0 = none
    size_t off_qop = 0, off_qconst = 0, off_tau = 0, off_prekeys = 0, off_lists = 0, off_parts = 0,
           off_mscratch = 0, bytes = 0;
    // thresholds seeded by counting on the tcgen05 path (run_counted_seed) instead of the list-keeping sample scan
    bool count = false;
    size_t off_uqimg = 0, off_uqconst = 0, off_seedpar = 0, off_seedhist = 0;
};

typedef void (*MmaKernel)(const mma::Params);

MmaKernel pick_mma_kernel(int C, bool fused, int warps) {
    if (warps == mma::WARPS_WIDE) {
        if (C == 1) return mma::scan_kernel<1, 1, 2, true, mma::WARPS_WIDE>;
        if (C == 2) return mma::scan_kernel<2, 1, 2, true, mma::WARPS_WIDE>;
        if (C == 3) return mma::scan_kernel<3, 1, 1, true, mma::WARPS_WIDE>;
        if (C == 4) return mma::scan_kernel<4, 1, 1, true, mma::WARPS_WIDE>;
        return nullptr;
    }
    if (warps == mma::WARPS_BATCH) {
        if (C == 1) return mma::scan_kernel<1, 2, 2, false, mma::WARPS_BATCH>;
        if (C == 2) return mma::scan_kernel<2, 2, 2, false, mma::WARPS_BATCH>;
        if (C == 3) return mma::scan_kernel<3, 1, 1, false, mma::WARPS_BATCH>;
        if (C == 4) return mma::scan_kernel<4, 1, 1, false, mma::WARPS_BATCH>;
        return nullptr;
    }
#define XFBQ_MMA_CASE(C_, MT_, NT_) \
    if (C == C_) return fused ? mma::scan_kernel<C_, MT_, NT_, true, mma::WARPS> : mma::scan_kernel<C_, MT_, NT_, false, mma::WARPS>;
    XFBQ_MMA_CASE(1, 2, 2) XFBQ_MMA_CASE(2, 2, 2) XFBQ_MMA_CASE(3, 1, 1) XFBQ_MMA_CASE(4, 1, 1)
#undef XFBQ_MMA_CASE
    return nullptr;
}

inline size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

void mma_shape(int64_t n, int wd, int C, int64_t nq, int k, const DeviceInfo &info, MmaShape *out) {
    const int sms = info.sms;
    MmaShape sh;
    sh.MT = C >= 3 ? 1 : 2;
    sh.NT = C >= 3 ? 1 : 2;
    if (nq <= 16 && env_int("XFBQ_NO_WIDE", 0) == 0 && env_int("XFBQ_NO_FUSED", 0) == 0) {
        sh.MT = 1;  // <= 16 queries: one 16-row tile, 16 warps per CTA
        sh.warps = mma::WARPS_WIDE;
    }
    sh.QPW = 16 * sh.MT;
    if ((nq + sh.QPW - 1) / sh.QPW >= mma::WARPS_BATCH && env_int("XFBQ_BATCH_WARPS", mma::WARPS_BATCH) == mma::WARPS_BATCH)
        sh.warps = mma::WARPS_BATCH;  // full batch: 12 query warps per CTA
    int cap = 64;
    while (cap < 2 * k) cap <<= 1;
    sh.cap = cap;
    const int64_t qwt = (nq + sh.QPW - 1) / sh.QPW;
    if (qwt >= sh.warps) {
        sh.QW = sh.warps; sh.DW = 1;
        sh.groups = static_cast<int>((qwt + sh.warps - 1) / sh.warps);
    } else {
        int qw = 1;
        while (qw < qwt) qw <<= 1;
        sh.QW = qw; sh.DW = sh.warps / qw; sh.groups = 1;
    }
    sh.nq_pad = static_cast<int64_t>(sh.groups) * sh.QW * sh.QPW;
    sh.n_pad = bundles_of(n) * 32;
    const int64_t stage_docs = static_cast<int64_t>(sh.warps) * 8 * sh.NT;
    sh.stages = (sh.n_pad + stage_docs - 1) / stage_docs;
    const int64_t W = static_cast<int64_t>(sh.groups) * sh.stages;
    int64_t grid = env_int("XFBQ_GRID", 0) > 0 ? env_int("XFBQ_GRID", 0) : sms;
    if (grid > W) grid = W;
    sh.grid = static_cast<int>(grid);
    // part slots: the largest number of CTA ranges [c*W/G, (c+1)*W/G) overlapping one group
    int slots = 1;
    for (int gr = 0; gr < sh.groups; ++gr) {
        const int64_t lo = static_cast<int64_t>(gr) * sh.stages, hi = lo + sh.stages;  // [lo, hi)
        int64_t c_first = lo * grid / W;
        while (c_first > 0 && c_first * W / grid > lo) --c_first;
        while ((c_first + 1) * W / grid <= lo) ++c_first;
        int64_t c_last = (hi - 1) * grid / W;
        while (c_last > 0 && c_last * W / grid > hi - 1) --c_last;
        while ((c_last + 1) * W / grid <= hi - 1) ++c_last;
        if (c_last - c_first + 1 > slots) slots = static_cast<int>(c_last - c_first + 1);
    }
    sh.slots = slots;
    sh.parts = slots * sh.DW;
    (void)wd;
    const int raw_stage = sh.warps * 8 * sh.NT * 64 * C;  // nibble layout: 64C bytes per document
    const int byte_stage = sh.warps * (sh.NT * C * 8) * 32 * 4;
    sh.fused = sh.QW == 1 && sh.groups == 1 && env_int("XFBQ_NO_FUSED", 0) == 0;
    int RR = env_int("XFBQ_RAW_STAGES", sh.fused ? (sh.warps == mma::WARPS ? 8 : 5) : (sh.warps == mma::WARPS ? 6 : 3)), BR = sh.fused ? 0 : env_int("XFBQ_BYTE_STAGES", sh.warps == mma::WARPS ? 4 : 3);
    const int br_min = sh.fused ? 0 : mma::AHEAD + 1;
    if (BR < br_min) BR = br_min;
    if (RR < 1) RR = 1;
    const size_t budget = static_cast<size_t>(info.smem_optin) - 1024;
    while (mma::smem_layout(raw_stage, byte_stage, RR, BR, cap, sh.warps).total > budget && RR > 2) --RR;
    while (mma::smem_layout(raw_stage, byte_stage, RR, BR, cap, sh.warps).total > budget && BR > br_min) --BR;
    while (mma::smem_layout(raw_stage, byte_stage, RR, BR, cap, sh.warps).total > budget && RR > 1) --RR;
    if (mma::smem_layout(raw_stage, byte_stage, RR, BR, cap, sh.warps).total > budget) RR = BR = 0;
    sh.RR = RR; sh.BR = BR;
    sh.smem = RR ? mma::smem_layout(raw_stage, byte_stage, RR, BR, cap, sh.warps).total : 0;
    sh.lists_bytes = static_cast<size_t>(sh.grid) * sh.warps * sh.QPW * cap * 8;
    sh.parts_bytes = static_cast<size_t>(sh.parts) * nq * k * 8;  // lists are emitted unsorted: always merged/sorted
    sh.mscratch_bytes = static_cast<size_t>(merge_scratch_parts(sh.parts, k, nq)) * nq * k * 8;
    *out = sh;
}

// Thresholds by counting (defined with the tcgen05 planning below; shared by both tensor engines).
int run_counted_seed(unsigned char *ws, const void *tiles, int64_t n, int64_t dim, int wd, const uint32_t *q, int64_t nq, int wq,
                     int k, int64_t sample, bool prep, size_t off_qimg, size_t off_qconst, size_t off_par, size_t off_hist,
                     int32_t *tau, cudaStream_t st, int32_t *theta0 = nullptr, uint32_t *ghist = nullptr);

int make_mma_plan(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k, bool have_nibbles, MmaPlan *plan, bool have_tiles = true) {
    MmaPlan pl;
    const int C = static_cast<int>(chunks128(dim));
    const char *eng = env_get("XFBQ_ENGINE");
    const bool forced_popc = eng && strcmp(eng, "popc") == 0;
    if (!have_nibbles || forced_popc || wd > 4 || wq > 7 || C < 1 || C > 4 || k > 1024 || nq < 1 || n < 1 ||
        env_int("XFBQ_FORCE_GENERIC", 0)) {
        *plan = pl;
        return XFBQ_OK;
    }
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    pl.ok = true;
    mma_shape(n, wd, C, nq, k, info, &pl.main);
    if (pl.main.RR == 0) {  // rings + sort scratch do not fit: leave it to the POPC engine
        pl.ok = false;
        *plan = pl;
        return XFBQ_OK;
    }
    // Small batches split the documents over every warp of the chip, so each candidate list sees
    // few documents and its own threshold tightens slowly; a sample scan of the first S documents
    // gives all of them a threshold of selectivity ~k/S up front.
    int64_t sample = env_int("XFBQ_SAMPLE", -1);
    // (Measured: for full batches the sample scan costs more than it saves -- every candidate list
    // of the sample scan floods from an open threshold -- so only small batches use it.)
    if (sample < 0) sample = pl.main.groups == 1 ? (nq <= 4 ? 32768 : 65536) : 131072;
    if (sample > 0 && (n < 16 * sample || sample < 4 * k)) sample = 0;
    pl.count = sample > 0 && have_tiles && env_int("XFBQ_SEED_HIST", 1) != 0;  // the counting seed reads byte tiles
    if (pl.count && sample > umma::SEED_MAX_SAMPLE(C)) sample = umma::SEED_MAX_SAMPLE(C);
    pl.sample = sample;
    if (sample && !pl.count) mma_shape(sample, wd, C, nq, k, info, &pl.pre);
    size_t off = 0;
    pl.off_qop = off; off = align256(off + static_cast<size_t>(pl.main.nq_pad) * 32 * C * 4);
    pl.off_qconst = off; off = align256(off + static_cast<size_t>(pl.main.nq_pad) * 4);
    pl.off_tau = off; off = align256(off + (sample ? static_cast<size_t>(nq) * 4 : 0));
    pl.off_prekeys = off; off = align256(off + (sample ? static_cast<size_t>(nq) * k * 8 : 0));
    pl.off_lists = off; off = align256(off + (pl.main.lists_bytes > pl.pre.lists_bytes ? pl.main.lists_bytes : pl.pre.lists_bytes));
    pl.off_parts = off; off = align256(off + (pl.main.parts_bytes > pl.pre.parts_bytes ? pl.main.parts_bytes : pl.pre.parts_bytes));
    pl.off_mscratch = off; off = align256(off + (pl.main.mscratch_bytes > pl.pre.mscratch_bytes ? pl.main.mscratch_bytes : pl.pre.mscratch_bytes));
    if (pl.count) {
        const int64_t uq = 128 * ((C >= 3 || nq <= 128) ? 1 : 2);  // queries per group of the counting kernel
        const int64_t nq_pad = (nq + uq - 1) / uq * uq;
        pl.off_uqimg = off; off = align256(off + static_cast<size_t>(nq_pad) * 128 * C);
        pl.off_uqconst = off; off = align256(off + static_cast<size_t>(nq_pad) * 4);
        pl.off_seedpar = off; off = align256(off + static_cast<size_t>(nq) * 8);
        pl.off_seedhist = off; off = align256(off + static_cast<size_t>(nq) * umma::SEED_BINS * 4);
    }
    pl.bytes = off;
    *plan = pl;
    return XFBQ_OK;
}

// One scan launch (+ merge of its part slots) over the first n documents of db.
int run_mma_scan(const MmaShape &sh, const MmaPlan &pl, unsigned char *ws, const void *nib, int64_t n, int C,
                 int64_t nq, int k, int64_t row_offset, const int32_t *tau_init, uint64_t *keys_out, cudaStream_t st) {
    MmaKernel kern = pick_mma_kernel(C, sh.fused, sh.warps);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sh.smem));
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "mma scan smem opt-in (%zu bytes): %s", sh.smem, cudaGetErrorString(e));
    mma::Params p;
    p.db = nib;
    p.n = n; p.n_pad = sh.n_pad; p.row_offset = row_offset;
    p.qop = reinterpret_cast<const uint32_t *>(ws + pl.off_qop);
    p.qconst = reinterpret_cast<const int32_t *>(ws + pl.off_qconst);
    p.tau_init = tau_init;
    p.lists = reinterpret_cast<uint64_t *>(ws + pl.off_lists);
    const bool direct = sh.parts == 1 && sh.cap <= mma::SORT_CAP_MAX;  // one sorted part: it is the result
    p.out = direct ? keys_out : reinterpret_cast<uint64_t *>(ws + pl.off_parts);
    p.nq = nq; p.stages = sh.stages; p.groups = sh.groups;
    p.k = k; p.cap = sh.cap; p.QW = sh.QW; p.DW = sh.DW;
    p.RR = sh.RR; p.BR = sh.BR;
    if (sh.slots > 1) {  // slots a group does not use stay KEY_INF
        e = cudaMemsetAsync(p.out, 0xFF, sh.parts_bytes, st);
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
    }
    const bool timed = g_timing && &sh == &pl.main;
    if (timed) timing_begin(st);
    kern<<<static_cast<unsigned>(sh.grid), sh.warps * 32, sh.smem, st>>>(p);
    if (timed) timing_end(st);
    if (int rc = check_launch("mma::scan_kernel")) return rc;
    if (direct) return XFBQ_OK;
    return launch_merge(p.out, sh.parts, nq, k, keys_out, reinterpret_cast<uint64_t *>(ws + pl.off_mscratch), st,
                        sh.cap > mma::SORT_CAP_MAX);  // large lists are emitted unsorted
}


// ----------------------------------------------------------------------------------------------
// Single-launch small-batch search (kernel in xfbq_coop.cuh): <= 16 queries, codes that fit a nibble, dim <= 512.
// ----------------------------------------------------------------------------------------------
struct CoopPlan {
    bool ok = false;
    int C = 1, cap = 0, RR = 0, grid = 0, seed_shift = 0, seed_offset = 0, hist_shift = 0, B = 0;
    int64_t stages = 0, seed_stride = 1;
    size_t smem = 0, off_qop = 0, off_qconst = 0, off_shist = 0, off_theta = 0, off_chist = 0, off_counts = 0, off_final = 0, off_lists = 0, bytes = 0;
    int final_cap = 0;
};

typedef void (*CoopKernel)(const coop::Params);
CoopKernel pick_coop_kernel(int C) {
    switch (C) {
        case 1: return coop::search_kernel<1>;
        case 2: return coop::search_kernel<2>;
        case 3: return coop::search_kernel<3>;
        case 4: return coop::search_kernel<4>;
    }
    return nullptr;
}

int make_coop_plan(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k, bool have_nibbles, CoopPlan *plan) {
    CoopPlan pl;
    *plan = pl;
    const int C = static_cast<int>(chunks128(dim));
    const char *eng = env_get("XFBQ_ENGINE");
    if (eng && *eng && strcmp(eng, "imma") != 0) return XFBQ_OK;  // part of the mma.sync engine
    if (!have_nibbles || wd > 4 || wq > 7 || C < 1 || C > 4 || k > 1024 || nq < 1 || nq > 16 || n < 1 || env_int("XFBQ_FORCE_GENERIC", 0) ||
        env_int("XFBQ_COOP", 1) == 0 || env_int("XFBQ_SAMPLE", -1) == 0)
        return XFBQ_OK;
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    static thread_local int coop_ok = -1;
    if (coop_ok < 0) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        coop_ok = (cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, dev) == cudaSuccess && v) ? 1 : 0;
    }
    if (!coop_ok) return XFBQ_OK;
    pl.C = C;
    pl.grid = info.sms > 148 ? 148 : info.sms;
    if (env_int("XFBQ_GRID", 0) > 0 && env_int("XFBQ_GRID", 0) < pl.grid) pl.grid = env_int("XFBQ_GRID", 0);
    const int NT = C <= 2 ? 2 : 1, TILE = 8 * NT;
    const int64_t n_pad = bundles_of(n) * 32;
    const int64_t sample_tiles = static_cast<int64_t>(pl.grid) * coop::WARPS * coop::SEED_TILES;
    const int64_t n_tiles = n_pad / TILE;
    if (n_tiles < 8 * sample_tiles || sample_tiles * TILE < 4 * static_cast<int64_t>(k)) return XFBQ_OK;  // small databases: the multi-launch path
    pl.seed_stride = n_tiles / sample_tiles;
    int cap = 64;
    while (cap < 2 * k) cap <<= 1;
    pl.cap = cap;
    const int stage_docs = coop::WARPS * TILE;
    pl.stages = (n_pad + stage_docs - 1) / stage_docs;
    if (pl.stages < pl.grid) return XFBQ_OK;
    const int raw_stage = stage_docs * 64 * C;
    int B = 8192;
    while (B < 4 * k) B <<= 1;
    const size_t budget = static_cast<size_t>(info.smem_optin) - 14 * 1024;  // static shared memory of the kernel (prefix sums, merge state)
    int RR = env_int("XFBQ_RAW_STAGES", 5);
    while (RR > 2 && mma::smem_layout(raw_stage, 0, RR, 0, cap, coop::WARPS).total > budget) --RR;
    if (mma::smem_layout(raw_stage, 0, RR, 0, cap, coop::WARPS).total > budget) return XFBQ_OK;
    while (B > 1024 && static_cast<size_t>(B) * 8 > static_cast<size_t>(RR) * raw_stage) B >>= 1;  // the merge buffer reuses the raw ring
    if (B < k + coop::WARPS * 32) return XFBQ_OK;
    pl.RR = RR; pl.B = B;
    pl.smem = mma::smem_layout(raw_stage, 0, RR, 0, cap, coop::WARPS).total;
    // sample histogram: SEED_BINS bins over the whole score range [-R, R]
    const int64_t R = xfbq_distance_upper_bound(dim, wd, wq);
    int shift = 0;
    while (((2 * R) >> shift) >= coop::SEED_BINS) ++shift;
    pl.seed_shift = shift; pl.seed_offset = static_cast<int>(R);
    int hs = 0;
    while ((static_cast<int64_t>(coop::CAND_BINS) << hs) < R / 56) ++hs;
    pl.hist_shift = env_int("XFBQ_UMMA_HIST_SHIFT", hs);
    size_t off = 0;
    pl.off_qop = off; off = align256(off + static_cast<size_t>(4 * C) * 32 * 16);
    pl.off_qconst = off; off = align256(off + 16 * 4);
    pl.off_shist = off; off = align256(off + static_cast<size_t>(16) * coop::SEED_BINS * 4);
    pl.off_theta = off; off = align256(off + 3 * 16 * 4);  // theta_g, theta0, row_bad
    pl.off_chist = off; off = align256(off + static_cast<size_t>(16) * coop::CAND_BINS * 4);
    pl.off_counts = off; off = align256(off + static_cast<size_t>(pl.grid) * coop::WARPS * 16 * 4);
    pl.final_cap = pl.B - coop::WARPS * 32;   // what one sort of the merge buffer takes
    pl.off_final = off; off = align256(off + 16 * 4 + static_cast<size_t>(16) * pl.final_cap * 8);
    pl.off_lists = off; off = align256(off + static_cast<size_t>(pl.grid) * coop::WARPS * 16 * cap * 8);
    pl.bytes = off;
    pl.ok = true;
    *plan = pl;
    return XFBQ_OK;
}

struct FloatQueries {  // float queries for the fused path (quantized inside the kernel), or all zero
    const void *x = nullptr;
    int f64 = 0;
    int64_t ld = 0;
    double scale = 1.0;
    uint64_t *nonfinite = nullptr;
    // k_select outputs (xfbq_kselect_small_*): candidates within `extra` of the k-th distance
    int extra = 0;
    uint64_t *cand_count = nullptr;
    int64_t *cand_ids = nullptr;
    int64_t cand_cap = 0;
    int *inexact = nullptr;
};

int run_coop(const CoopPlan &cp, unsigned char *ws, const void *nib, int64_t n, int64_t dim, int wd, const uint32_t *q, int64_t nq, int wq,
             int k, int64_t row_offset, uint64_t *keys_out, cudaStream_t st, const FloatQueries &fq = FloatQueries()) {
    CoopKernel kern = pick_coop_kernel(cp.C);
    if (!kern) return fail(XFBQ_E_UNSUPPORTED, "no single-launch kernel for C=%d", cp.C);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cp.smem));
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "single-launch search smem opt-in (%zu bytes): %s", cp.smem, cudaGetErrorString(e));
    coop::Params p;
    p.nib = nib;
    p.n = n; p.n_pad = bundles_of(n) * 32; p.row_offset = row_offset;
    p.q = q; p.nq = static_cast<int>(nq); p.wq = wq; p.wd = wd; p.dim = static_cast<int>(dim);
    p.xq = fq.x; p.xq_f64 = fq.f64; p.ldq = fq.ld; p.scale = fq.scale;
    p.nonfinite = reinterpret_cast<unsigned long long *>(fq.nonfinite);
    p.row_bad = reinterpret_cast<int *>(ws + cp.off_theta) + 32;
    p.extra = fq.extra;
    p.cand_count = reinterpret_cast<unsigned long long *>(fq.cand_count);
    p.cand_ids = fq.cand_ids; p.cand_cap = fq.cand_cap; p.inexact = fq.inexact;
    p.qop = reinterpret_cast<uint32_t *>(ws + cp.off_qop);
    p.qconst = reinterpret_cast<int32_t *>(ws + cp.off_qconst);
    p.shist = reinterpret_cast<uint32_t *>(ws + cp.off_shist);
    p.theta_g = reinterpret_cast<int32_t *>(ws + cp.off_theta);
    p.theta0 = p.theta_g + 16;
    p.chist = reinterpret_cast<uint32_t *>(ws + cp.off_chist);
    p.lists = reinterpret_cast<uint64_t *>(ws + cp.off_lists);
    p.counts = reinterpret_cast<int *>(ws + cp.off_counts);
    p.final_cnt = reinterpret_cast<unsigned *>(ws + cp.off_final);
    p.final_list = reinterpret_cast<uint64_t *>(ws + cp.off_final + 64);
    p.final_cap = cp.final_cap;
    p.keys_out = keys_out;
    p.stages = cp.stages; p.seed_tile_stride = cp.seed_stride;
    p.k = k; p.cap = cp.cap; p.RR = cp.RR;
    p.seed_shift = cp.seed_shift; p.seed_offset = cp.seed_offset; p.hist_shift = cp.hist_shift; p.merge_B = cp.B;
    p.prof = g_prof;
    void *args[] = {&p};
    if (g_timing) timing_begin(st);
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern), dim3(static_cast<unsigned>(cp.grid)), dim3(coop::WARPS * 32), args, cp.smem, st);
    if (g_timing) timing_end(st);
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "coop::search_kernel: %s", cudaGetErrorString(e));
    return check_launch("coop::search_kernel");
}

// ----------------------------------------------------------------------------------------------
// tcgen05 engine planning (kernel in xfbq_umma.cuh).
// ----------------------------------------------------------------------------------------------
struct UmmaShape {
    int MT = 2, DW = 1, groups = 1, grid = 1, slots = 1, parts = 1, cap = 0, NS = 0;
    int C = 1, KP = 1;   // chunks of 128 dims per operand stage, K parts per tile
    bool queue = false;  // scan_queue_kernel (main scans) vs scan_kernel (sample scans: open thresholds)
    bool direct = false; // queue kernel with one work item per CTA: lists stay in place, the bounded merge reads them (no emission)
    bool count = false;  // sample scan that only counts scores into per-query histograms (scan_kernel<.., SEED = true>)
    int64_t tile_stride = 1, n_valid = 0;  // counting scan: stage i reads tile i * tile_stride of a database of n_valid documents
    int ring_rows = 64;
    int n_seg = 1, seg_stages = 0;  // queue kernel: document slices (= partial results per query) and stages per slice
    int64_t stages = 0, nq_pad = 0, n_pad = 0;
    size_t smem = 0, lists_bytes = 0, parts_bytes = 0, mscratch_bytes = 0;
};

struct UmmaPlan {
    bool ok = false;
    UmmaShape main, pre;
    int64_t sample = 0;
    size_t off_qimg = 0, off_qconst = 0, off_tau = 0, off_prekeys = 0, off_lists = 0, off_parts = 0, off_mscratch = 0,
           off_theta0 = 0, off_ghist = 0, off_seedpar = 0, off_seedhist = 0, off_counts = 0, bytes = 0;
};

typedef void (*UmmaKernel)(const umma::Params);

UmmaKernel pick_umma_kernel(int C, int MT, bool queue, bool count = false, bool direct = false, int KP = 1) {
    if (KP == 2) {  // 513..1024 dims: two K parts of 3 or 4 chunks, one query tile
        if (MT != 1 || (C != 3 && C != 4)) return nullptr;
        if (count) return C == 3 ? umma::scan_kernel<3, 1, true, 2> : umma::scan_kernel<4, 1, true, 2>;
        if (queue && direct) return C == 3 ? umma::scan_queue_kernel<3, 1, true, 2> : umma::scan_queue_kernel<4, 1, true, 2>;
        if (queue) return C == 3 ? umma::scan_queue_kernel<3, 1, false, 2> : umma::scan_queue_kernel<4, 1, false, 2>;
        return C == 3 ? umma::scan_kernel<3, 1, false, 2> : umma::scan_kernel<4, 1, false, 2>;
    }
    if (queue && direct) {
        if (C == 1) return MT == 2 ? umma::scan_queue_kernel<1, 2, true> : umma::scan_queue_kernel<1, 1, true>;
        if (C == 2) return MT == 2 ? umma::scan_queue_kernel<2, 2, true> : umma::scan_queue_kernel<2, 1, true>;
        if (C == 3 && MT == 1) return umma::scan_queue_kernel<3, 1, true>;
        if (C == 4 && MT == 1) return umma::scan_queue_kernel<4, 1, true>;
        return nullptr;
    }
    if (count) {
        if (C == 1) return MT == 2 ? umma::scan_kernel<1, 2, true> : umma::scan_kernel<1, 1, true>;
        if (C == 2) return MT == 2 ? umma::scan_kernel<2, 2, true> : umma::scan_kernel<2, 1, true>;
        if (C == 3 && MT == 1) return umma::scan_kernel<3, 1, true>;
        if (C == 4 && MT == 1) return umma::scan_kernel<4, 1, true>;
        return nullptr;
    }
    if (queue) {
        if (C == 1) return MT == 2 ? umma::scan_queue_kernel<1, 2> : umma::scan_queue_kernel<1, 1>;
        if (C == 2) return MT == 2 ? umma::scan_queue_kernel<2, 2> : umma::scan_queue_kernel<2, 1>;
        if (C == 3 && MT == 1) return umma::scan_queue_kernel<3, 1>;
        if (C == 4 && MT == 1) return umma::scan_queue_kernel<4, 1>;
        return nullptr;
    }
    if (C == 1) return MT == 2 ? umma::scan_kernel<1, 2> : umma::scan_kernel<1, 1>;
    if (C == 2) return MT == 2 ? umma::scan_kernel<2, 2> : umma::scan_kernel<2, 1>;
    if (C == 3 && MT == 1) return umma::scan_kernel<3, 1>;
    if (C == 4 && MT == 1) return umma::scan_kernel<4, 1>;
    return nullptr;
}

void umma_shape(int64_t n, int C, int64_t nq, int k, int MT, const DeviceInfo &info, UmmaShape *out, bool seed_scan = false,
                bool allow_queue = true, bool count = false, int KP = 1) {
    UmmaShape sh;
    sh.MT = MT;
    sh.C = C; sh.KP = KP;
    sh.count = count;
    sh.queue = !seed_scan && allow_queue && env_int("XFBQ_UMMA_QUEUE", 1) != 0;
    sh.DW = (MT == 2 || sh.queue) ? 1 : 2;
    int cap = 64;
    while (cap < 2 * k) cap <<= 1;
    if (sh.queue) {  // resolver-owned lists: a compaction costs a resolver ~cap/32 steps, so let lists run longer
        const int want = env_int("XFBQ_UMMA_CAP", 0);
        if (want >= k + 40) cap = (want + 7) & ~7;
    }
    sh.cap = cap;
    const int64_t qpg = 128 * MT;
    sh.groups = static_cast<int>((nq + qpg - 1) / qpg);
    sh.nq_pad = static_cast<int64_t>(sh.groups) * qpg;
    sh.n_pad = bundles_of(n) * 32;
    sh.stages = (sh.n_pad + umma::STAGE_DOCS - 1) / umma::STAGE_DOCS;
    const int64_t W = static_cast<int64_t>(sh.groups) * sh.stages;
    int64_t grid = env_int("XFBQ_GRID", 0) > 0 ? env_int("XFBQ_GRID", 0) : info.sms;
    // (The sample scan runs on every SM too: capping it at a few CTAs per query group saved list start-ups but
    // left most of the chip idle for small batches -- 256 queries: 1.7 ms on 4 CTAs.)
    if (seed_scan && env_int("XFBQ_SEED_SPLIT", 0) > 0 && env_int("XFBQ_GRID", 0) <= 0) {
        const int64_t cap_grid = static_cast<int64_t>(sh.groups) * env_int("XFBQ_SEED_SPLIT", 0);
        if (grid > cap_grid) grid = cap_grid;
    }
    if (grid > W) grid = W;
    sh.grid = static_cast<int>(grid);
    int slots = 1;
    for (int gr = 0; gr < sh.groups; ++gr) {
        const int64_t lo = static_cast<int64_t>(gr) * sh.stages, hi = lo + sh.stages;
        int64_t c_first = lo * grid / W;
        while (c_first > 0 && c_first * W / grid > lo) --c_first;
        while ((c_first + 1) * W / grid <= lo) ++c_first;
        int64_t c_last = (hi - 1) * grid / W;
        while (c_last > 0 && c_last * W / grid > hi - 1) --c_last;
        while ((c_last + 1) * W / grid <= hi - 1) ++c_last;
        if (c_last - c_first + 1 > slots) slots = static_cast<int>(c_last - c_first + 1);
    }
    if (sh.queue) {
        // Work items = document slices x query groups, dealt to the CTAs round-robin (umma::Items).  Pick the
        // slice count that fills whole waves of CTAs; slices stay long enough to amortise the per-item list
        // start-up and emission.
        int64_t min_stages = env_int("XFBQ_UMMA_MIN_SLICE", 512);
        // Few query groups over a mid-size database: slices of 512 tiles would leave SMs without work (one group over 4M rows:
        // 61 slices on 148 SMs, the scan at 4.6 TB/s instead of > 7).  Filling the first wave matters more than the per-slice
        // list work there: slices may shrink to what one wave needs, down to 32 tiles (4 096 documents; 1M x 256, 256 queries:
        // 61 slices 0.304 ms, 148 slices 0.251).
        const int64_t fill_S = (grid + sh.groups - 1) / sh.groups;
        if (sh.stages / min_stages < fill_S && env_int("XFBQ_UMMA_FILL", 1) != 0) {
            const int64_t floor_stages = env_int("XFBQ_UMMA_FILL_FLOOR", 32);
            const int64_t relaxed = sh.stages / fill_S > floor_stages ? sh.stages / fill_S : floor_stages;
            if (relaxed < min_stages) min_stages = relaxed;
        }
        int best = 1;
        double best_score = -1.0;
        for (int S = 1; S <= 256; ++S) {
            if (S > 1 && (sh.stages + S - 1) / S < min_stages) break;
            const int64_t items = static_cast<int64_t>(S) * sh.groups;
            const int64_t waves = (items + grid - 1) / grid;
            // fill of the waves, minus the per-slice list work, minus a little per extra wave (a single wave also merges
            // its lists in place; 1 250 queries: 29 slices x 5 groups in one wave 2.11 ms, 59 x 5 in two waves 2.17-2.19)
            const double score = static_cast<double>(items) / static_cast<double>(waves * grid) - 0.0005 * S - 0.01 * static_cast<double>(waves - 1);
            if (score > best_score) { best_score = score; best = S; }
        }
        if (env_int("XFBQ_UMMA_SLICES", 0) > 0) best = env_int("XFBQ_UMMA_SLICES", 0);
        if (best > sh.stages) best = static_cast<int>(sh.stages);
        sh.n_seg = best;
        sh.seg_stages = static_cast<int>((sh.stages + best - 1) / best);
        sh.n_seg = static_cast<int>((sh.stages + sh.seg_stages - 1) / sh.seg_stages);  // no empty slices
        const int64_t items = static_cast<int64_t>(sh.n_seg) * sh.groups;
        if (sh.grid > items) sh.grid = static_cast<int>(items);
        slots = sh.n_seg;
        sh.direct = items <= sh.grid && sh.n_seg > 1 && sh.n_seg <= 256 && env_int("XFBQ_UMMA_DIRECT", 1) != 0 && env_int("XFBQ_MERGE_BOUNDED", 1) != 0 &&
                    env_int("XFBQ_UMMA_SHARE", 1) != 0;
    }
    sh.slots = slots;
    sh.parts = slots * sh.DW;
    int NS = env_int("XFBQ_UMMA_STAGES", 5);
    const size_t budget = static_cast<size_t>(info.smem_optin);
    auto smem_need = [&](int ns) { return static_cast<size_t>(sh.queue ? umma::q_smem_layout(C, ns, sh.ring_rows).total : umma::smem_layout(C, MT, ns, sh.count).total); };
    if (sh.queue && smem_need(NS < 3 ? NS : 3) > budget) sh.ring_rows = 32;  // wide documents: shorter rings rather than fewer than three tiles in flight
    while (NS > 2 && smem_need(NS) > budget) --NS;
    sh.NS = smem_need(NS) <= budget ? NS : 0;
    sh.smem = smem_need(NS);
    sh.lists_bytes = static_cast<size_t>(sh.grid) * umma::EPI_WARPS * 32 * cap * 8;
    sh.parts_bytes = static_cast<size_t>(sh.parts) * nq * k * 8;
    sh.mscratch_bytes = static_cast<size_t>(merge_scratch_parts(sh.parts, k, nq)) * nq * k * 8;
    if (count) sh.lists_bytes = sh.parts_bytes = sh.mscratch_bytes = 0;  // the counting scan keeps no lists
    *out = sh;
}

int make_umma_plan(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k, bool have_nibbles, UmmaPlan *plan) {
    UmmaPlan pl;
    *plan = pl;
    const TileGeom tg = tile_geom(dim);
    const int C = tg.Cp, KP = tg.KP;
    const char *eng = env_get("XFBQ_ENGINE");
    if (eng && *eng && strcmp(eng, "umma") != 0) return XFBQ_OK;  // another engine was asked for
    const bool forced = eng && strcmp(eng, "umma") == 0;
    if (!have_nibbles || wq > 7 || tg.CP < 1 || tg.CP > 8 || k > 1024 || n < 1 || env_int("XFBQ_FORCE_GENERIC", 0))  // any document width: the B operand is u8
        return XFBQ_OK;
    // where the mma.sync engine cannot go (codes wider than a nibble, more than 512 dims) this engine also takes the small
    // batches, single queries included: the POPC kernels pay 1 POPC per code byte and query (one query over 8M x 768:
    // 3.60 ms there, 0.97 ms here; 4M x 1024: 2.39 / 1.06; 1M x 768: 0.56 / 0.42 -- profiles/wide_single_r2c.log)
    const bool no_imma = wd > 4 || tg.CP > 4;
    if (!forced && nq < env_int("XFBQ_UMMA_MIN_NQ", no_imma ? 1 : 17)) return XFBQ_OK;  // <= 16 queries: the mma.sync scans (HBM-bound on the nibble layout; a 24-query batch took 0.72 ms there, 0.55 ms here)
    if (nq < 1) return XFBQ_OK;
    if (merge_group_max(k) == 0 || nq > 65535) return XFBQ_OK;  // lists are emitted unsorted: needs the tree merge
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    const int MT = (C >= 3 || KP == 2 || nq <= 128) ? 1 : 2;
    // Sample scan that seeds the thresholds (measured on 10M x 256, 10k queries: 16k documents split over at
    // most 4 CTAs per query group balance its cost -- it starts from open lists -- against the rows the main
    // scan's resolvers then have to handle).
    int64_t sample = env_int("XFBQ_SAMPLE", -1);
    if (sample < 0) {
        sample = 16384;
        while (sample < 64 * static_cast<int64_t>(k)) sample <<= 1;
        // small databases: a smaller sample still seeds the thresholds (and with them the queue kernel) as long as it holds 64 k documents
        if (env_int("XFBQ_SAMPLE_SHRINK", 1))
            while (sample > 4096 && n < 8 * sample && (sample >> 1) >= 64 * static_cast<int64_t>(k)) sample >>= 1;
    }
    if (sample > 0 && (n < 8 * sample || sample < 4 * k)) sample = 0;
    // Without seeded thresholds every score passes at first: list work dominates and the kernel whose eight
    // epilogue warps own their lists beats the two resolvers of the queue kernel (100k x 128, 100 queries: 4x).
    // With seeded thresholds the queue kernel wins at every size that was measured (profiles/queue_min_ab2_r2d.log: 150k-1M
    // rows, 32-1 024 queries, 1.6-9x; the list-keeping kernel was the choice below 2M rows until the counted seed, the
    // bounded merge and the first-wave fill of the slice planner existed).
    const int64_t groups = (nq + 128 * MT - 1) / (128 * MT);
    const bool big = n >= env_int("XFBQ_UMMA_QUEUE_MIN_N", 1) || groups >= 16;
    umma_shape(n, C, nq, k, MT, info, &pl.main, false, sample > 0 && big, false, KP);
    if (pl.main.NS == 0) return XFBQ_OK;
    pl.sample = sample;
    // Queue-kernel scans are seeded by counting (histogram of the sample's scores, no lists); the list-keeping
    // sample scan remains for XFBQ_SEED_HIST=0.  A counted sample is nearly free, so it can be larger.
    const bool count = sample > 0 && pl.main.queue && env_int("XFBQ_SEED_HIST", 1) != 0;
    if (count) {
        if (env_int("XFBQ_SAMPLE", -1) < 0) {
            // a counted sample may be 1/8 of the database; what it saves grows with k (list insertions ~ k ln(n / sample)).
            // Measured per 10k queries: top-100 over 2.5M rows 5.41 ms with 64k documents, 5.05 with 128k; 1.25M rows 4.51 ms
            // with 16k, 3.61 with 64k, 3.38 with 128k; 1M x 128: 3.53 ms with 32k, 3.27 with 64k; top-10 over 1.2M rows 2.35 ms
            // with 64k, 2.26 with 32k.
            const int64_t cap_k = k >= 64 ? 131072 : (k >= 16 ? 65536 : 32768);
            while (sample < cap_k && n >= 16 * sample) sample <<= 1;
        }
        if (sample > umma::SEED_MAX_SAMPLE(C)) sample = umma::SEED_MAX_SAMPLE(C);
        pl.sample = sample;
    }
    if (sample) umma_shape(sample, C, nq, k, MT, info, &pl.pre, true, true, count, KP);
    if (sample && pl.pre.NS == 0) return XFBQ_OK;
    if (count && pl.main.stages < 2 * pl.pre.stages) return XFBQ_OK;  // (cannot happen: n >= 16 * sample) sampled tiles must be full tiles
    if (count) {  // the counted sample is spread over the whole database (every stride-th tile)
        pl.pre.tile_stride = env_int("XFBQ_SEED_SPREAD", 1) ? pl.main.stages / pl.pre.stages : 1;
        if (pl.pre.tile_stride < 1) pl.pre.tile_stride = 1;
        pl.pre.n_valid = n;
    }
    size_t off = 0;
    pl.off_qimg = off; off = align256(off + static_cast<size_t>(pl.main.nq_pad) * 128 * tg.CT);
    pl.off_qconst = off; off = align256(off + static_cast<size_t>(pl.main.nq_pad) * 4);
    pl.off_tau = off; off = align256(off + (sample ? static_cast<size_t>(nq) * 4 : 0));
    pl.off_prekeys = off; off = align256(off + (sample ? static_cast<size_t>(nq) * k * 8 : 0));
    pl.off_lists = off; off = align256(off + (pl.main.lists_bytes > pl.pre.lists_bytes ? pl.main.lists_bytes : pl.pre.lists_bytes));
    pl.off_parts = off; off = align256(off + (pl.main.parts_bytes > pl.pre.parts_bytes ? pl.main.parts_bytes : pl.pre.parts_bytes));
    pl.off_mscratch = off; off = align256(off + (pl.main.mscratch_bytes > pl.pre.mscratch_bytes ? pl.main.mscratch_bytes : pl.pre.mscratch_bytes));
    const bool use_hist = pl.main.queue && sample > 0 && env_int("XFBQ_UMMA_HIST", 1) != 0;
    pl.off_theta0 = off; off = align256(off + (use_hist ? static_cast<size_t>(nq) * 4 : 0));
    pl.off_ghist = off; off = align256(off + (use_hist ? static_cast<size_t>(nq) * umma::HIST_BINS * 4 : 0));
    pl.off_seedpar = off; off = align256(off + (count ? static_cast<size_t>(nq) * 8 : 0));
    pl.off_seedhist = off; off = align256(off + (count ? static_cast<size_t>(nq) * umma::SEED_BINS * 4 : 0));
    if (!(sample > 0)) pl.main.direct = false;  // the bounded merge needs the seeded, shared thresholds
    pl.off_counts = off; off = align256(off + (pl.main.direct ? static_cast<size_t>(pl.main.grid) * 128 * pl.main.MT * 4 : 0));
    pl.bytes = off;
    pl.ok = true;
    *plan = pl;
    return XFBQ_OK;
}

// z with P(N(0,1) > z) = p, by bisection on erfc (host side, once per call)
double normal_quantile(double p) {
    if (p >= 0.5) return 0.0;
    double lo = 0.0, hi = 8.0;
    for (int i = 0; i < 60; ++i) {
        const double mid = 0.5 * (lo + hi);
        if (0.5 * erfc(mid / 1.4142135623730951) > p) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

int run_umma_scan(const UmmaShape &sh, const UmmaPlan &pl, unsigned char *ws, const void *nib, int64_t n, int C,
                  int64_t nq, int k, int64_t row_offset, const int32_t *tau_init, uint64_t *keys_out, cudaStream_t st) {
    const bool direct = sh.direct && &sh == &pl.main && tau_init != nullptr;
    (void)C;
    UmmaKernel kern = pick_umma_kernel(sh.C, sh.MT, sh.queue, sh.count, direct, sh.KP);
    if (!kern) return fail(XFBQ_E_UNSUPPORTED, "no tcgen05 kernel for C=%d MT=%d KP=%d", sh.C, sh.MT, sh.KP);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sh.smem));
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "umma scan smem opt-in (%zu bytes): %s", sh.smem, cudaGetErrorString(e));
    umma::Params p;
    p.db = nib;  // byte tiles (the caller passes the tile region of the derived buffer)
    p.n = sh.count ? sh.n_valid : n; p.n_pad = sh.n_pad; p.row_offset = row_offset;
    p.tile_stride = sh.count ? sh.tile_stride : 1;
    p.qimg = ws + pl.off_qimg;
    p.qconst = reinterpret_cast<const int32_t *>(ws + pl.off_qconst);
    p.tau_init = tau_init;
    p.theta_g = (tau_init && env_int("XFBQ_UMMA_SHARE", 1)) ? const_cast<int32_t *>(tau_init) : nullptr;  // the seeded thresholds double as the shared ones
    p.lists = reinterpret_cast<uint64_t *>(ws + pl.off_lists);
    p.out = reinterpret_cast<uint64_t *>(ws + pl.off_parts);
    p.nq = nq; p.stages = sh.stages; p.groups = sh.groups;
    p.k = k; p.cap = sh.cap; p.NS = sh.NS;
    p.n_seg = sh.n_seg; p.seg_stages = sh.seg_stages; p.ring_rows = sh.ring_rows;
    const bool use_hist = sh.queue && tau_init && pl.off_ghist > pl.off_theta0;
    p.ghist = use_hist ? reinterpret_cast<uint32_t *>(ws + pl.off_ghist) : nullptr;
    p.theta0 = use_hist ? reinterpret_cast<const int32_t *>(ws + pl.off_theta0) : nullptr;
    p.hist_shift = g_hist_shift;
    p.seed_par = sh.count ? reinterpret_cast<const int2 *>(ws + pl.off_seedpar) : nullptr;
    p.seed_hist = sh.count ? reinterpret_cast<uint32_t *>(ws + pl.off_seedhist) : nullptr;
    p.list_counts = direct ? reinterpret_cast<int *>(ws + pl.off_counts) : nullptr;
    p.prof = (&sh == &pl.main) ? g_prof : nullptr;
    p.pace = 48;
#ifdef XFBQ_DEBUG_KNOBS  // timing experiments only (results are NOT valid under them): compiled out of the shipped library
    p.debug = env_int("XFBQ_UMMA_DEBUG", 0);
#else
    p.debug = 0;
#endif
    if (sh.slots > 1 && !sh.queue && !sh.count) {  // slots a group does not use stay KEY_INF (the queue kernel writes every slice)
        e = cudaMemsetAsync(p.out, 0xFF, sh.parts_bytes, st);
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
    }
    const bool timed = g_timing && &sh == &pl.main;
    if (timed) timing_begin(st);
    kern<<<static_cast<unsigned>(sh.grid), sh.queue ? umma::Q_THREADS : umma::THREADS, sh.smem, st>>>(p);
    if (timed) timing_end(st);
    if (int rc = check_launch("umma::scan_kernel")) return rc;
    if (sh.count) return XFBQ_OK;  // histograms only: seed_bounds_kernel follows
    if (p.theta_g && sh.parts > 1 && env_int("XFBQ_MERGE_BOUNDED", 1)) {
        int B = 512;
        while (B < 4 * k) B <<= 1;  // k <= 1024 on this engine: at most 8192 keys = 64 KB
        int threads = B / 4 > 512 ? 512 : B / 4;
        const int want = env_int("XFBQ_MERGE_BUF", 0);  // tests: a small buffer forces the overflow path (power of two >= k + threads)
        if (want >= k + threads && (want & (want - 1)) == 0) B = want;
        const size_t smem = static_cast<size_t>(B) * 8;
        if (smem > 48 * 1024) {
            e = cudaFuncSetAttribute(merge_bounded_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "merge smem opt-in: %s", cudaGetErrorString(e));
        }
        if (direct) {
            ListSrc src;
            src.counts = p.list_counts; src.nq_cta = 128 * sh.MT; src.cap = sh.cap; src.groups = sh.groups;
            merge_bounded_kernel<<<static_cast<unsigned>(nq), threads, smem, st>>>(p.lists, sh.parts, nq, k, B, p.theta_g, p.qconst, keys_out, src);
        } else {
            merge_bounded_kernel<<<static_cast<unsigned>(nq), threads, smem, st>>>(p.out, sh.parts, nq, k, B, p.theta_g, p.qconst, keys_out);
        }
        return check_launch("merge_bounded_kernel");
    }
    return launch_merge(p.out, sh.parts, nq, k, keys_out, reinterpret_cast<uint64_t *>(ws + pl.off_mscratch), st, true);
}

// Thresholds by counting: frame per query from 128 sampled scores, 64-bin histogram of the whole sample on the
// tensor cores (every stride-th byte tile of the database), threshold = lower edge of the bin where the suffix
// count reaches k.  tau[q] is in the accumulator domain both tensor engines use (Dq - distance).
int run_counted_seed(unsigned char *ws, const void *tiles, int64_t n, int64_t dim, int wd, const uint32_t *q, int64_t nq, int wq,
                     int k, int64_t sample, bool prep, size_t off_qimg, size_t off_qconst, size_t off_par, size_t off_hist,
                     int32_t *tau, cudaStream_t st, int32_t *theta0, uint32_t *ghist) {
    const TileGeom tg = tile_geom(dim);
    const int C = tg.Cp;
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    const int MT = (C >= 3 || tg.KP == 2 || nq <= 128) ? 1 : 2;
    UmmaPlan pl;
    umma_shape(sample, C, nq, k, MT, info, &pl.pre, true, true, true, tg.KP);
    const int64_t total_stages = (bundles_of(n) * 32 + umma::STAGE_DOCS - 1) / umma::STAGE_DOCS;
    if (pl.pre.NS == 0 || total_stages < 2 * pl.pre.stages)
        return fail(XFBQ_E_UNSUPPORTED, "counted seed: sample %lld does not fit n=%lld dim=%lld", (long long)sample, (long long)n, (long long)dim);
    pl.pre.tile_stride = env_int("XFBQ_SEED_SPREAD", 1) ? total_stages / pl.pre.stages : 1;
    pl.pre.n_valid = n;
    pl.off_qimg = off_qimg; pl.off_qconst = off_qconst; pl.off_seedpar = off_par; pl.off_seedhist = off_hist;
    unsigned char *qimg = ws + off_qimg;
    if (prep) {
        umma::prep_queries_kernel<<<static_cast<unsigned>((pl.pre.nq_pad * 32 + 255) / 256), 256, 0, st>>>(
            q, nq, pl.pre.nq_pad, static_cast<int>(dim), wq, wd, tg.CT, MT, qimg, reinterpret_cast<int32_t *>(ws + off_qconst));
        if (int rc = check_launch("umma::prep_queries_kernel")) return rc;
    }
    int2 *par = reinterpret_cast<int2 *>(ws + off_par);
    uint32_t *hist = reinterpret_cast<uint32_t *>(ws + off_hist);
    umma::seed_stats_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(static_cast<const unsigned char *>(tiles), qimg, nq, tg.CT, pl.pre.stages, pl.pre.tile_stride,
                                                                    static_cast<float>(normal_quantile(static_cast<double>(k) / static_cast<double>(sample))),
                                                                    0.25f * env_int("XFBQ_SEED_BELOW4", 8), par, hist);
    if (int rc = check_launch("umma::seed_stats_kernel")) return rc;
    if (int rc = run_umma_scan(pl.pre, pl, ws, tiles, sample, C, nq, k, 0, nullptr, nullptr, st)) return rc;
    umma::seed_bounds_kernel<<<static_cast<unsigned>((nq * 32 + 255) / 256), 256, 0, st>>>(hist, par, nq, k, tau, theta0, ghist);
    return check_launch("umma::seed_bounds_kernel");
}

int run_umma(const UmmaPlan &up, unsigned char *ws, const void *nib, int64_t n, int64_t dim, int wd, const uint32_t *q,
             int64_t nq, int wq, int k, int64_t row_offset, uint64_t *keys_out, cudaStream_t st) {
    const int C = up.main.C;
    unsigned char *qimg = ws + up.off_qimg;
    int32_t *qconst = reinterpret_cast<int32_t *>(ws + up.off_qconst);
    umma::prep_queries_kernel<<<static_cast<unsigned>((up.main.nq_pad * 32 + 255) / 256), 256, 0, st>>>(
        q, nq, up.main.nq_pad, static_cast<int>(dim), wq, wd, tile_geom(dim).CT, up.main.MT, qimg, qconst);
    if (int rc = check_launch("umma::prep_queries_kernel")) return rc;
    const int32_t *tau_init = nullptr;
    if (up.sample) {
        uint64_t *prekeys = reinterpret_cast<uint64_t *>(ws + up.off_prekeys);
        int32_t *tau = reinterpret_cast<int32_t *>(ws + up.off_tau);
        const bool hist_main = up.off_ghist > up.off_theta0;  // global candidate histogram of the main scan, bins measured from the seeded thresholds
        if (up.pre.count) {   // the bounds kernel also copies the thresholds and clears the main scan's histogram
            if (int rc = run_counted_seed(ws, nib, n, dim, wd, q, nq, wq, k, up.sample, false, up.off_qimg, up.off_qconst, up.off_seedpar,
                                          up.off_seedhist, tau, st, hist_main ? reinterpret_cast<int32_t *>(ws + up.off_theta0) : nullptr,
                                          hist_main ? reinterpret_cast<uint32_t *>(ws + up.off_ghist) : nullptr)) return rc;
        } else {
            if (int rc = run_umma_scan(up.pre, up, ws, nib, up.sample, C, nq, k, row_offset, nullptr, prekeys, st)) return rc;
            mma::tau_from_keys_kernel<<<static_cast<unsigned>((nq + 255) / 256), 256, 0, st>>>(prekeys, qconst, nq, k, tau);
            if (int rc = check_launch("tau_from_keys_kernel")) return rc;
        }
        tau_init = tau;
        if (hist_main) {
            if (!up.pre.count) {
                cudaError_t e = cudaMemcpyAsync(ws + up.off_theta0, tau, static_cast<size_t>(nq) * 4, cudaMemcpyDeviceToDevice, st);
                if (e == cudaSuccess) e = cudaMemsetAsync(ws + up.off_ghist, 0, static_cast<size_t>(nq) * umma::HIST_BINS * 4, st);
                if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "histogram setup: %s", cudaGetErrorString(e));
            }
            // scores of interest lie within ~1/64 of the distance range below the seed: 256 bins of width 2^shift cover it
            const int64_t ub = xfbq_distance_upper_bound(dim, wd, wq);
            int shift = 0;
            while ((static_cast<int64_t>(umma::HIST_BINS) << shift) < ub / 56) ++shift;
            g_hist_shift = env_int("XFBQ_UMMA_HIST_SHIFT", shift);
        }
#ifdef XFBQ_DEBUG_KNOBS
        if (env_int("XFBQ_DEBUG_TAU_NEVER", 0)) cudaMemsetAsync(tau, 0x40, static_cast<size_t>(nq) * 4, st);  // timing experiments only: nothing passes
#endif
    }
    return run_umma_scan(up.main, up, ws, nib, n, C, nq, k, row_offset, tau_init, keys_out, st);
}

template <typename T>
int quantize_pack_impl(const T *x, int64_t n, int64_t dim, int64_t ld, double scale, int width,
                       void *out, uint64_t *nonfinite, void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (!(scale > 0.0)) return fail(XFBQ_E_INVALID, "scale must be positive, got %g", scale);
    if (n < 0 || dim < 1 || ld < dim) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld ld=%lld", (long long)n, (long long)dim, (long long)ld);
    if (dim > (1 << 20)) return fail(XFBQ_E_UNSUPPORTED, "dim %lld too large", (long long)dim);
    if (n == 0) return XFBQ_OK;
    if (!x || !out || !nonfinite) return fail(XFBQ_E_INVALID, "null pointer");
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    const int64_t nb = bundles_of(n);
    if (sizeof(T) == 4 && dim % 4 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        scale * 2147483648.0 <= 1e30 && scale * 2147483648.0 >= 1e-30 && env_int("XFBQ_QUANT_SLOW", 0) == 0) {
        const int64_t units = nb * chunks128(dim) * 4;
        int64_t fblocks = (units + 7) / 8;
        const int64_t fmax = static_cast<int64_t>(info.sms) * 16;
        if (fblocks > fmax) fblocks = fmax;
        typedef void (*FastKernel)(const float *, int64_t, int, int64_t, double, int, uint32_t *, unsigned long long *);
        static const FastKernel kernels[XFBQ_MAX_WIDTH] = {
            quantize_pack_f32_fast_kernel<1>, quantize_pack_f32_fast_kernel<2>, quantize_pack_f32_fast_kernel<3>,
            quantize_pack_f32_fast_kernel<4>, quantize_pack_f32_fast_kernel<5>, quantize_pack_f32_fast_kernel<6>,
            quantize_pack_f32_fast_kernel<7>, quantize_pack_f32_fast_kernel<8>};
        kernels[width - 1]<<<static_cast<unsigned>(fblocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const float *>(x), n, static_cast<int>(dim), ld, scale, static_cast<int>(chunks128(dim)),
            static_cast<uint32_t *>(out), reinterpret_cast<unsigned long long *>(nonfinite));
        return check_launch("quantize_pack_f32_fast_kernel");
    }
    int64_t blocks = (nb + QP_WARPS - 1) / QP_WARPS;
    const int64_t max_blocks = static_cast<int64_t>(info.sms) * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    quantize_pack_kernel<T><<<static_cast<unsigned>(blocks), QP_WARPS * 32, 0, static_cast<cudaStream_t>(stream)>>>(
        x, n, static_cast<int>(dim), ld, scale, width, static_cast<int>(chunks128(dim)),
        static_cast<uint4 *>(out), reinterpret_cast<unsigned long long *>(nonfinite));
    return check_launch("quantize_pack_kernel");
}

template <typename T>
int quantize_queries_impl(const T *x, int64_t nq, int64_t dim, int64_t ld, double scale, int width,
                          uint32_t *out, uint64_t *nonfinite, void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (!(scale > 0.0)) return fail(XFBQ_E_INVALID, "scale must be positive, got %g", scale);
    if (nq < 0 || dim < 1 || ld < dim) return fail(XFBQ_E_INVALID, "bad shape nq=%lld dim=%lld ld=%lld", (long long)nq, (long long)dim, (long long)ld);
    if (dim > (1 << 20)) return fail(XFBQ_E_UNSUPPORTED, "dim %lld too large", (long long)dim);
    if (nq == 0) return XFBQ_OK;
    if (!x || !out || !nonfinite) return fail(XFBQ_E_INVALID, "null pointer");
    const int64_t blocks = (nq * 32 + 255) / 256;
    quantize_queries_kernel<T><<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, nq, static_cast<int>(dim), ld, scale, width, static_cast<int>(chunks128(dim)), out,
        reinterpret_cast<unsigned long long *>(nonfinite));
    return check_launch("quantize_queries_kernel");
}

}  // namespace

// ------------------------------------------------------------------------------------- C ABI
XFBQ_API int xfbq_abi_version(void) { return XFBQ_ABI_VERSION; }
XFBQ_API const char *xfbq_last_error(void) { return g_err; }
XFBQ_API int xfbq_set_timing(int enable) {
    if (enable && !g_evs[0][0]) {
        for (int i = 0; i < TIMING_PAIRS; ++i)
            if (cudaEventCreate(&g_evs[i][0]) != cudaSuccess || cudaEventCreate(&g_evs[i][1]) != cudaSuccess)
                return fail(XFBQ_E_CUDA, "cudaEventCreate failed");
    }
    g_timing = enable != 0;
    g_ev_count = 0;
    return XFBQ_OK;
}

XFBQ_API int xfbq_debug_profile(void *device_counters) {
    g_prof = static_cast<unsigned long long *>(device_counters);
    return XFBQ_OK;
}

XFBQ_API int xfbq_last_scan_ms(float *ms_out) {
    if (!ms_out) return fail(XFBQ_E_INVALID, "null pointer");
    if (g_ev_count == 0) return fail(XFBQ_E_INVALID, "no timed scan recorded (call xfbq_set_timing(1) first)");
    cudaEvent_t *pair = g_evs[(g_ev_count - 1) % TIMING_PAIRS];
    cudaError_t e = cudaEventSynchronize(pair[1]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms_out, pair[0], pair[1]);
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "event timing: %s", cudaGetErrorString(e));
    return XFBQ_OK;
}

XFBQ_API int xfbq_scan_ms_mean(float *mean_ms_out, int *launches_out) {
    if (!mean_ms_out || !launches_out) return fail(XFBQ_E_INVALID, "null pointer");
    if (g_ev_count == 0) return fail(XFBQ_E_INVALID, "no timed scan recorded (call xfbq_set_timing(1) first)");
    const int kept = g_ev_count < TIMING_PAIRS ? g_ev_count : TIMING_PAIRS;
    double sum = 0.0;
    for (int i = 0; i < kept; ++i) {
        cudaEvent_t *pair = g_evs[(g_ev_count - 1 - i) % TIMING_PAIRS];
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(pair[1]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, pair[0], pair[1]);
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "event timing: %s", cudaGetErrorString(e));
        sum += ms;
    }
    *mean_ms_out = static_cast<float>(sum / kept);
    *launches_out = kept;
    return XFBQ_OK;
}

XFBQ_API int64_t xfbq_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
XFBQ_API int64_t xfbq_chunks128(int64_t dim) { return chunks128(dim); }

XFBQ_API int64_t xfbq_db_bytes(int64_t n, int64_t dim, int width) {
    return bundles_of(n) * width * chunks128(dim) * 32 * 16;
}

XFBQ_API int64_t xfbq_query_bytes(int64_t nq, int64_t dim, int width) {
    return nq * width * chunks128(dim) * 16;
}

XFBQ_API int64_t xfbq_distance_upper_bound(int64_t dim, int wx, int wy) {
    return dim * static_cast<int64_t>((1 << wx) - 1) * static_cast<int64_t>((1 << wy) - 1);
}

XFBQ_API int xfbq_quantize_pack_f32(const float *x, int64_t n, int64_t dim, int64_t ld, double scale,
                                    int width, void *out, uint64_t *nonfinite, void *stream) {
    return quantize_pack_impl<float>(x, n, dim, ld, scale, width, out, nonfinite, stream);
}

XFBQ_API int xfbq_quantize_pack_f64(const double *x, int64_t n, int64_t dim, int64_t ld, double scale,
                                    int width, void *out, uint64_t *nonfinite, void *stream) {
    return quantize_pack_impl<double>(x, n, dim, ld, scale, width, out, nonfinite, stream);
}

XFBQ_API int xfbq_quantize_queries_f32(const float *q, int64_t nq, int64_t dim, int64_t ld, double scale,
                                       int width, uint32_t *out, uint64_t *nonfinite, void *stream) {
    return quantize_queries_impl<float>(q, nq, dim, ld, scale, width, out, nonfinite, stream);
}

XFBQ_API int xfbq_quantize_queries_f64(const double *q, int64_t nq, int64_t dim, int64_t ld, double scale,
                                       int width, uint32_t *out, uint64_t *nonfinite, void *stream) {
    return quantize_queries_impl<double>(q, nq, dim, ld, scale, width, out, nonfinite, stream);
}

XFBQ_API int xfbq_planes_to_bundles(const uint64_t *planes, int64_t n, int64_t dim, int width, void *out,
                                    void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0) return XFBQ_OK;
    if (!planes || !out) return fail(XFBQ_E_INVALID, "null pointer");
    const int C = static_cast<int>(chunks128(dim));
    const int64_t total = bundles_of(n) * width * C * 32;
    planes_to_bundles_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        planes, n, static_cast<int>((dim + 63) / 64), width, C, static_cast<uint4 *>(out), total);
    return check_launch("planes_to_bundles_kernel");
}

XFBQ_API int xfbq_bundles_to_planes(const void *db, int64_t n, int64_t dim, int width, uint64_t *planes,
                                    void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0) return XFBQ_OK;
    if (!planes || !db) return fail(XFBQ_E_INVALID, "null pointer");
    const int C = static_cast<int>(chunks128(dim));
    const int64_t total = bundles_of(n) * width * C * 32;
    bundles_to_planes_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4 *>(db), n, static_cast<int>((dim + 63) / 64), width, C, planes, total);
    return check_launch("bundles_to_planes_kernel");
}

// Derived layouts of one index, in one buffer: [nibble layout][byte tiles].
inline int64_t nibble_region_bytes(int64_t n, int64_t dim, int wd = 4) {
    if (wd > 4 || chunks128(dim) > 4) return 0;  // no mma.sync engine for these: the derived buffer holds the byte tiles only
    return ((bundles_of(n) * 32 * chunks128(dim) * 64 + 1023) / 1024) * 1024;
}
inline int64_t tile_count(int64_t n) { return (n + umma::STAGE_DOCS - 1) / umma::STAGE_DOCS; }
inline bool tiles_supported(int64_t dim) { const int64_t C = chunks128(dim); return C >= 1 && C <= 8; }

XFBQ_API int64_t xfbq_derived_bytes(int64_t n, int64_t dim, int width) {
    return nibble_region_bytes(n, dim, width) + xfbq_tile_region_bytes(n, dim);
}
XFBQ_API int64_t xfbq_nibble_bytes(int64_t n, int64_t dim) { return xfbq_derived_bytes(n, dim, 4); }

XFBQ_API int64_t xfbq_nibble_region_bytes(int64_t n, int64_t dim, int width) { return nibble_region_bytes(n, dim, width); }
XFBQ_API int64_t xfbq_tile_region_bytes(int64_t n, int64_t dim) {
    return tiles_supported(dim) ? tile_count(n) * umma::STAGE_DOCS * tile_geom(dim).CT * 128 : 0;
}

XFBQ_API int xfbq_build_nibbles(const void *db, int64_t n, int64_t dim, int width, void *out, void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0 || nibble_region_bytes(n, dim, width) == 0) return XFBQ_OK;
    if (!db || !out) return fail(XFBQ_E_INVALID, "null pointer");
    const int C = static_cast<int>(chunks128(dim));
    const int64_t n_pad = bundles_of(n) * 32, total = n_pad * 4 * C;
    mma::planes_to_nibbles_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint32_t *>(db), n_pad, width, C, static_cast<uint4 *>(out));
    return check_launch("planes_to_nibbles_kernel");
}

XFBQ_API int xfbq_build_tiles(const void *db, int64_t n, int64_t dim, int width, void *out, void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0 || !tiles_supported(dim)) return XFBQ_OK;
    if (!db || !out) return fail(XFBQ_E_INVALID, "null pointer");
    const int C = static_cast<int>(chunks128(dim)), CT = tile_geom(dim).CT;
    const int64_t n_pad = bundles_of(n) * 32;
    const int64_t tiles = tile_count(n), groups = tiles * umma::STAGE_DOCS * 4 * CT;
    umma::planes_to_tiles_kernel<<<static_cast<unsigned>((groups + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint32_t *>(db), n_pad, tiles, width, C, CT, static_cast<unsigned char *>(out));
    return check_launch("planes_to_tiles_kernel");
}

XFBQ_API int xfbq_restore_codes_from_nibbles(const void *nibbles, int64_t n, int64_t dim, int width, void *db_out, void *stream) {
    if (width < 1 || width > 4) return fail(XFBQ_E_UNSUPPORTED, "nibble layout holds codes of at most 4 bits, got %d", width);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0) return XFBQ_OK;
    if (nibble_region_bytes(n, dim, width) == 0) return fail(XFBQ_E_UNSUPPORTED, "no nibble layout for dim=%lld", (long long)dim);
    if (!nibbles || !db_out) return fail(XFBQ_E_INVALID, "null pointer");
    const int C = static_cast<int>(chunks128(dim));
    const int64_t n_pad = bundles_of(n) * 32, total = n_pad * 4 * C;
    mma::nibbles_to_planes_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4 *>(nibbles), n_pad, width, C, static_cast<uint32_t *>(db_out));
    return check_launch("nibbles_to_planes_kernel");
}

XFBQ_API int xfbq_restore_codes_from_tiles(const void *tiles, int64_t n, int64_t dim, int width, void *db_out, void *stream) {
    if (!width_ok(width)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d", width);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0) return XFBQ_OK;
    if (!tiles_supported(dim)) return fail(XFBQ_E_UNSUPPORTED, "no tile layout for dim=%lld", (long long)dim);
    if (!tiles || !db_out) return fail(XFBQ_E_INVALID, "null pointer");
    const int C = static_cast<int>(chunks128(dim)), CT = tile_geom(dim).CT;
    const int64_t n_pad = bundles_of(n) * 32, total = n_pad * 4 * C;
    umma::tiles_to_planes_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const unsigned char *>(tiles), n_pad, width, C, CT, static_cast<uint32_t *>(db_out));
    return check_launch("tiles_to_planes_kernel");
}

XFBQ_API int xfbq_build_derived(const void *db, int64_t n, int64_t dim, int width, void *out, void *stream) {
    if (int rc = xfbq_build_nibbles(db, n, dim, width, out, stream)) return rc;
    if (n <= 0 || dim < 1 || !out) return XFBQ_OK;
    return xfbq_build_tiles(db, n, dim, width, static_cast<unsigned char *>(out) + nibble_region_bytes(n, dim, width), stream);
}

XFBQ_API int xfbq_planes_to_nibbles(const void *db, int64_t n, int64_t dim, int width, void *nib_out, void *stream) {
    if (width < 1 || width > 4) return fail(XFBQ_E_UNSUPPORTED, "nibble layout holds codes of at most 4 bits, got %d", width);
    return xfbq_build_derived(db, n, dim, width, nib_out, stream);
}

XFBQ_API int xfbq_batch_distances(const void *db, int64_t n, int64_t dim, int wd, const uint32_t *q, int wq,
                                  uint64_t *out, void *stream) {
    if (!width_ok(wd) || !width_ok(wq)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d/%d", wd, wq);
    if (n < 0 || dim < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld", (long long)n, (long long)dim);
    if (n == 0) return XFBQ_OK;
    if (!db || !q || !out) return fail(XFBQ_E_INVALID, "null pointer");
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    const int C = static_cast<int>(chunks128(dim));
    const size_t smem = static_cast<size_t>(wq) * C * 16;
    if (smem > 48 * 1024) return fail(XFBQ_E_UNSUPPORTED, "dim %lld too large for batch_distances", (long long)dim);
    int64_t blocks = (bundles_of(n) + 7) / 8;
    const int64_t max_blocks = static_cast<int64_t>(info.sms) * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    batch_distances_kernel<<<static_cast<unsigned>(blocks), 256, smem, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4 *>(db), n, wd, C, q, wq, out);
    return check_launch("batch_distances_kernel");
}

XFBQ_API int xfbq_collect_candidates(const void *db, int64_t n, int64_t dim, int wd, const uint32_t *q, int wq,
                                     int64_t threshold, int64_t *ids_out, int64_t cap, uint64_t *count_out, void *stream) {
    if (!width_ok(wd) || !width_ok(wq)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d/%d", wd, wq);
    if (n < 0 || dim < 1 || cap < 0) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld cap=%lld", (long long)n, (long long)dim, (long long)cap);
    if (!count_out) return fail(XFBQ_E_INVALID, "null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(count_out, 0, 8, st);
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
    if (n == 0 || threshold < 0) return XFBQ_OK;
    if (!db || !q) return fail(XFBQ_E_INVALID, "null pointer");
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    const int C = static_cast<int>(chunks128(dim));
    const size_t smem = static_cast<size_t>(wq) * C * 16;
    if (smem > 48 * 1024) return fail(XFBQ_E_UNSUPPORTED, "dim %lld too large for collect_candidates", (long long)dim);
    int64_t blocks = (bundles_of(n) + 7) / 8;
    const int64_t max_blocks = static_cast<int64_t>(info.sms) * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    const uint32_t thr = threshold > 0xFFFFFFFFll ? 0xFFFFFFFFu : static_cast<uint32_t>(threshold);
    typedef void (*FastKernel)(const uint4 *, int64_t, const uint32_t *, uint32_t, int64_t *, int64_t, unsigned long long *);
    FastKernel fast = nullptr;
#define XFBQ_CASE(WD_, WQ_, C_) if (wd == WD_ && wq == WQ_ && C == C_) fast = collect_candidates_fast_kernel<WD_, WQ_, C_>;
    XFBQ_CASE(3, 4, 1) XFBQ_CASE(3, 4, 2) XFBQ_CASE(3, 4, 4)
    XFBQ_CASE(4, 4, 1) XFBQ_CASE(4, 4, 2) XFBQ_CASE(4, 4, 4)
#undef XFBQ_CASE
    if (fast && !env_int("XFBQ_FORCE_GENERIC", 0)) {
        fast<<<static_cast<unsigned>(blocks), 256, 0, st>>>(static_cast<const uint4 *>(db), n, q, thr, ids_out, ids_out ? cap : 0,
                                                            reinterpret_cast<unsigned long long *>(count_out));
        return check_launch("collect_candidates_fast_kernel");
    }
    collect_candidates_kernel<<<static_cast<unsigned>(blocks), 256, smem, st>>>(
        static_cast<const uint4 *>(db), n, wd, C, q, wq, thr, ids_out, ids_out ? cap : 0, reinterpret_cast<unsigned long long *>(count_out));
    return check_launch("collect_candidates_kernel");
}


namespace {

template <typename T>
int abs_order_stats_impl(const T *x, int64_t count, int64_t rank_lo, int64_t rank_hi, void *ws, int64_t ws_bytes, T *out2,
                         uint64_t *nan_count, void *stream) {
    if (count < 1) return fail(XFBQ_E_INVALID, "cannot take order statistics of an empty array");
    if (rank_lo < 0 || rank_hi < rank_lo || rank_hi >= count)
        return fail(XFBQ_E_INVALID, "bad ranks %lld, %lld for %lld elements", (long long)rank_lo, (long long)rank_hi, (long long)count);
    if (!x || !ws || !out2 || !nan_count) return fail(XFBQ_E_INVALID, "null pointer");
    if (ws_bytes < static_cast<int64_t>(sizeof(sel::State))) return fail(XFBQ_E_INVALID, "workspace too small: need %zu bytes", sizeof(sel::State));
    if ((reinterpret_cast<uintptr_t>(ws) & 7) != 0) return fail(XFBQ_E_INVALID, "workspace must be 8-byte aligned");
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    sel::State *state = static_cast<sel::State *>(ws);
    sel::init_state_kernel<<<1, 256, 0, st>>>(state, rank_lo, rank_hi);
    if (int rc = check_launch("sel::init_state_kernel")) return rc;
    const size_t smem = static_cast<size_t>(sel::COPIES) * sel::BINS * 4;
    cudaError_t e = cudaFuncSetAttribute(sel::hist_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(sel::hist_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "select smem opt-in: %s", cudaGetErrorString(e));
    constexpr int V = 16 / sizeof(T);
    int64_t blocks = (count / V + 255) / 256;
    const int64_t max_blocks = static_cast<int64_t>(info.sms) * 3;  // 64 KB of histogram copies per block: three blocks per SM
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    int hi_bit = static_cast<int>(sizeof(T)) * 8;
    bool first = true;
    while (hi_bit > 0) {
        const int nbits = hi_bit >= sel::DIGIT_BITS ? sel::DIGIT_BITS : hi_bit;
        const int lo_bit = hi_bit - nbits;
        if (first) sel::hist_kernel<T, true><<<static_cast<unsigned>(blocks), 256, smem, st>>>(x, count, lo_bit, nbits, state);
        else sel::hist_kernel<T, false><<<static_cast<unsigned>(blocks), 256, smem, st>>>(x, count, lo_bit, nbits, state);
        if (int rc = check_launch("sel::hist_kernel")) return rc;
        sel::pick_kernel<<<1, 1024, 0, st>>>(state, nbits);
        if (int rc = check_launch("sel::pick_kernel")) return rc;
        hi_bit = lo_bit;
        first = false;
    }
    sel::finish_kernel<T><<<1, 32, 0, st>>>(state, out2, reinterpret_cast<unsigned long long *>(nan_count));
    return check_launch("sel::finish_kernel");
}

int refine_k2(int k) {
    int K2 = 256;
    while (K2 < k) K2 <<= 1;
    return K2;
}
int refine_blocks(int64_t count, int sms) {
    int64_t g = (count + 8191) / 8192;
    if (g > 2 * static_cast<int64_t>(sms)) g = 2 * sms;
    return g < 1 ? 1 : static_cast<int>(g);
}

template <typename T>
int refine_impl(const T *rows, int64_t n, int64_t dim, int64_t ld, int gathered, const int64_t *ids, int64_t count, const double *q, int k,
                double *sims_out, int64_t *ids_out, void *ws, int64_t ws_bytes, void *stream) {
    if (n < 0 || dim < 1 || ld < dim || count < 0) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld ld=%lld count=%lld", (long long)n, (long long)dim, (long long)ld, (long long)count);
    if (k < 1) return fail(XFBQ_E_INVALID, "k must be >= 1, got %d", k);
    if (k > XFBQ_MAX_K) return fail(XFBQ_E_UNSUPPORTED, "k=%d exceeds XFBQ_MAX_K=%d", k, XFBQ_MAX_K);
    if (!sims_out || !ids_out) return fail(XFBQ_E_INVALID, "null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    if (!rows || !ids || !q || !ws) return fail(XFBQ_E_INVALID, "null pointer");
    const int G = refine_blocks(count, info.sms);
    const int64_t need = xfbq_refine_workspace_bytes(count, k);
    if (ws_bytes < need) return fail(XFBQ_E_INVALID, "workspace too small: need %lld bytes, got %lld", (long long)need, (long long)ws_bytes);
    double *sims = static_cast<double *>(ws);
    sel::RankPair *part = reinterpret_cast<sel::RankPair *>(static_cast<unsigned char *>(ws) + align256(static_cast<size_t>(count) * 8));
    if (count > 0) {
        sel::gather_dot_kernel<T><<<static_cast<unsigned>((count * 32 + 255) / 256), 256, 0, st>>>(rows, ld, static_cast<int>(dim), gathered ? nullptr : ids, count, q, sims);
        if (int rc = check_launch("sel::gather_dot_kernel")) return rc;
    }
    const int K2 = refine_k2(k);
    const size_t smem = static_cast<size_t>(2) * K2 * sizeof(sel::RankPair);
    cudaError_t e = cudaFuncSetAttribute(sel::rank_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(sel::rank_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "refine smem opt-in: %s", cudaGetErrorString(e));
    sel::rank_partial_kernel<<<static_cast<unsigned>(G), 256, smem, st>>>(sims, ids, count, k, K2, part);
    if (int rc = check_launch("sel::rank_partial_kernel")) return rc;
    sel::rank_final_kernel<<<1, 256, smem, st>>>(part, static_cast<int64_t>(G) * k, k, K2, sims_out, ids_out);
    return check_launch("sel::rank_final_kernel");
}

}  // namespace

XFBQ_API int64_t xfbq_select_workspace_bytes(void) { return static_cast<int64_t>(align256(sizeof(sel::State))); }

XFBQ_API int xfbq_abs_order_stats_f32(const float *x, int64_t count, int64_t rank_lo, int64_t rank_hi, void *ws, int64_t ws_bytes,
                                      float *out2, uint64_t *nan_count, void *stream) {
    return abs_order_stats_impl<float>(x, count, rank_lo, rank_hi, ws, ws_bytes, out2, nan_count, stream);
}

XFBQ_API int xfbq_abs_order_stats_f64(const double *x, int64_t count, int64_t rank_lo, int64_t rank_hi, void *ws, int64_t ws_bytes,
                                      double *out2, uint64_t *nan_count, void *stream) {
    return abs_order_stats_impl<double>(x, count, rank_lo, rank_hi, ws, ws_bytes, out2, nan_count, stream);
}

XFBQ_API int64_t xfbq_refine_workspace_bytes(int64_t count, int k) {
    if (count < 0 || k < 1) return -1;
    DeviceInfo info;
    int sms = 148;
    if (device_info(&info) == XFBQ_OK) sms = info.sms;
    return static_cast<int64_t>(align256(static_cast<size_t>(count) * 8) +
                                align256(static_cast<size_t>(refine_blocks(count, sms)) * k * sizeof(sel::RankPair)));
}

XFBQ_API int xfbq_refine_f32(const float *rows, int64_t n, int64_t dim, int64_t ld, int gathered, const int64_t *ids, int64_t count, const double *q, int k,
                             double *sims_out, int64_t *ids_out, void *ws, int64_t ws_bytes, void *stream) {
    return refine_impl<float>(rows, n, dim, ld, gathered, ids, count, q, k, sims_out, ids_out, ws, ws_bytes, stream);
}

XFBQ_API int xfbq_collect_candidates_nibbles(const void *nib, int64_t n, int64_t dim, int wd, const uint32_t *q, int wq,
                                             int64_t threshold, int64_t *ids_out, int64_t cap, uint64_t *count_out, void *stream) {
    if (!width_ok(wd) || !width_ok(wq)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d/%d", wd, wq);
    if (n < 0 || dim < 1 || cap < 0) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld cap=%lld", (long long)n, (long long)dim, (long long)cap);
    const int C = static_cast<int>(chunks128(dim));
    if (wd > 4 || wq > 7 || C > 4) return fail(XFBQ_E_UNSUPPORTED, "no nibble layout for doc_bits=%d query_bits=%d dim=%lld", wd, wq, (long long)dim);
    if (!count_out) return fail(XFBQ_E_INVALID, "null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(count_out, 0, 8, st);
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
    if (n == 0 || threshold < 0) return XFBQ_OK;
    if (!nib || !q) return fail(XFBQ_E_INVALID, "null pointer");
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    int64_t blocks = (n + 255) / 256;
    const int64_t max_blocks = static_cast<int64_t>(info.sms) * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    const uint32_t thr = threshold > 0xFFFFFFFFll ? 0xFFFFFFFFu : static_cast<uint32_t>(threshold);
    typedef void (*Kern)(const uint4 *, int64_t, int, int, const uint32_t *, int, uint32_t, int64_t *, int64_t, unsigned long long *);
    static const Kern kernels[4] = {sel::collect_candidates_nib_warp_kernel<1>, sel::collect_candidates_nib_warp_kernel<2>,
                                    sel::collect_candidates_nib_kernel<3>, sel::collect_candidates_nib_warp_kernel<4>};
    blocks = (bundles_of(n) + 7) / 8;   // a warp per bundle of 32 documents
    if (blocks > max_blocks) blocks = max_blocks;
    kernels[C - 1]<<<static_cast<unsigned>(blocks), 256, 0, st>>>(static_cast<const uint4 *>(nib), n, static_cast<int>(dim), wd, q, wq, thr, ids_out,
                                                                  ids_out ? cap : 0, reinterpret_cast<unsigned long long *>(count_out));
    return check_launch("sel::collect_candidates_nib_kernel");
}

XFBQ_API int xfbq_distance_histogram(const int64_t *dist, int64_t n, int64_t bins, uint64_t *hist, uint64_t *out_of_range, void *stream) {
    if (n < 0 || bins < 1) return fail(XFBQ_E_INVALID, "bad shape n=%lld bins=%lld", (long long)n, (long long)bins);
    if (!hist || !out_of_range) return fail(XFBQ_E_INVALID, "null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(hist, 0, static_cast<size_t>(bins) * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(out_of_range, 0, 8, st);
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
    if (n == 0) return XFBQ_OK;
    if (!dist) return fail(XFBQ_E_INVALID, "null pointer");
    DeviceInfo info;
    if (int rc = device_info(&info)) return rc;
    int64_t blocks = (n + 255) / 256;
    if (blocks > static_cast<int64_t>(info.sms) * 8) blocks = static_cast<int64_t>(info.sms) * 8;
    sel::dist_histogram_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(dist, n, bins, reinterpret_cast<unsigned long long *>(hist),
                                                                             reinterpret_cast<unsigned long long *>(out_of_range));
    return check_launch("sel::dist_histogram_kernel");
}

XFBQ_API int xfbq_histogram_kth(const uint64_t *hist, int64_t bins, int64_t k, int64_t *kth_out, void *stream) {
    if (bins < 1 || k < 1) return fail(XFBQ_E_INVALID, "bad arguments bins=%lld k=%lld", (long long)bins, (long long)k);
    if (!hist || !kth_out) return fail(XFBQ_E_INVALID, "null pointer");
    sel::hist_kth_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const unsigned long long *>(hist), bins,
                                                                           static_cast<unsigned long long>(k), reinterpret_cast<long long *>(kth_out));
    return check_launch("sel::hist_kth_kernel");
}

XFBQ_API int64_t xfbq_gather_workspace_bytes(int64_t n) {
    if (n < 0) return -1;
    return static_cast<int64_t>(align256((static_cast<size_t>((n + 65535) / 65536) + 2) * 8));
}

XFBQ_API int xfbq_gather_le_count(const int64_t *dist, int64_t n, int64_t threshold, void *workspace, int64_t workspace_bytes, void *stream) {
    if (n < 0) return fail(XFBQ_E_INVALID, "negative n");
    if (!workspace || workspace_bytes < xfbq_gather_workspace_bytes(n)) return fail(XFBQ_E_INVALID, "workspace too small");
    const int blocks = static_cast<int>((n + 65535) / 65536);
    unsigned long long *counts = static_cast<unsigned long long *>(workspace);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (blocks == 0) {
        cudaError_t e = cudaMemsetAsync(counts, 0, 16, st);
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
        return XFBQ_OK;
    }
    if (!dist) return fail(XFBQ_E_INVALID, "null pointer");
    sel::count_le_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(dist, n, threshold, 65536, counts);
    if (int rc = check_launch("sel::count_le_kernel")) return rc;
    sel::exclusive_scan_kernel<<<1, 1024, 0, st>>>(counts, blocks);   // counts[blocks] = total
    return check_launch("sel::exclusive_scan_kernel");
}

XFBQ_API int xfbq_gather_le_ids(const int64_t *dist, int64_t n, int64_t threshold, const void *workspace, int64_t *ids_out, void *stream) {
    if (n < 0) return fail(XFBQ_E_INVALID, "negative n");
    if (n == 0) return XFBQ_OK;
    if (!dist || !workspace || !ids_out) return fail(XFBQ_E_INVALID, "null pointer");
    const int blocks = static_cast<int>((n + 65535) / 65536);
    sel::gather_le_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        dist, n, threshold, 65536, static_cast<const unsigned long long *>(workspace), ids_out);
    return check_launch("sel::gather_le_kernel");
}


namespace {
int search_small_impl(const void *db, const void *nib, int64_t n, int64_t dim, int wd, const void *queries, int f64, int64_t nq, int64_t ld,
                      double scale, int wq, int k, int64_t row_offset, uint64_t *keys_out, uint64_t *nonfinite, void *workspace,
                      int64_t workspace_bytes, void *stream, int64_t extra = 0, uint64_t *cand_count = nullptr, int64_t *cand_ids = nullptr,
                      int64_t cand_cap = 0, int *inexact = nullptr) {
    if (extra < 0 || extra >= (1ll << 30)) return fail(XFBQ_E_INVALID, "extra distance out of range");
    if (cand_count && !inexact) return fail(XFBQ_E_INVALID, "null pointer");
    if (!width_ok(wd) || !width_ok(wq)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d/%d", wd, wq);
    if (!(scale > 0.0)) return fail(XFBQ_E_INVALID, "scale must be positive, got %g", scale);
    if (n < 1 || dim < 1 || nq < 1 || ld < dim) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld nq=%lld ld=%lld", (long long)n, (long long)dim, (long long)nq, (long long)ld);
    if (k < 1) return fail(XFBQ_E_INVALID, "k must be >= 1, got %d", k);
    if (row_offset < 0 || row_offset + n > (1ll << 32)) return fail(XFBQ_E_UNSUPPORTED, "row ids must fit 32 bits");
    (void)db;  // the single-launch search reads the nibble layout only: the packed codes may have been released (null)
    if (!nib || !queries || !keys_out || !nonfinite || !workspace) return fail(XFBQ_E_INVALID, "null pointer");
    CoopPlan cp;
    if (int rc = make_coop_plan(n, dim, wd, nq, wq, k, true, &cp)) return rc;
    if (!cp.ok) return fail(XFBQ_E_UNSUPPORTED, "no single-launch search for this shape (xfbq_search_small_workspace_bytes returns 0)");
    if (workspace_bytes < static_cast<int64_t>(cp.bytes))
        return fail(XFBQ_E_INVALID, "workspace too small: need %zu bytes, got %lld", cp.bytes, (long long)workspace_bytes);
    FloatQueries fq;
    fq.x = queries; fq.f64 = f64; fq.ld = ld; fq.scale = scale; fq.nonfinite = nonfinite;
    fq.extra = static_cast<int>(extra); fq.cand_count = cand_count; fq.cand_ids = cand_ids; fq.cand_cap = cand_cap; fq.inexact = inexact;
    return run_coop(cp, static_cast<unsigned char *>(workspace), nib, n, dim, wd, nullptr, nq, wq, k, row_offset, keys_out,
                    static_cast<cudaStream_t>(stream), fq);
}
}  // namespace

XFBQ_API int64_t xfbq_search_small_workspace_bytes(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k) {
    if (!width_ok(wd) || !width_ok(wq) || n < 1 || dim < 1 || nq < 1 || k < 1 || k > XFBQ_MAX_K) return 0;
    CoopPlan cp;
    if (make_coop_plan(n, dim, wd, nq, wq, k, true, &cp) || !cp.ok) return 0;
    return static_cast<int64_t>(cp.bytes);
}

XFBQ_API int xfbq_search_small_f32(const void *db, const void *nib, int64_t n, int64_t dim, int wd, const float *queries, int64_t nq, int64_t ld,
                                   double scale, int wq, int k, int64_t row_offset, uint64_t *keys_out, uint64_t *nonfinite, void *workspace,
                                   int64_t workspace_bytes, void *stream) {
    return search_small_impl(db, nib, n, dim, wd, queries, 0, nq, ld, scale, wq, k, row_offset, keys_out, nonfinite, workspace, workspace_bytes, stream);
}

XFBQ_API int xfbq_search_small_f64(const void *db, const void *nib, int64_t n, int64_t dim, int wd, const double *queries, int64_t nq, int64_t ld,
                                   double scale, int wq, int k, int64_t row_offset, uint64_t *keys_out, uint64_t *nonfinite, void *workspace,
                                   int64_t workspace_bytes, void *stream) {
    return search_small_impl(db, nib, n, dim, wd, queries, 1, nq, ld, scale, wq, k, row_offset, keys_out, nonfinite, workspace, workspace_bytes, stream);
}

namespace {
// `layouts` argument of the planning calls: 0 = no derived layout, XFBQ_LAYOUT_NIBBLES | XFBQ_LAYOUT_TILES, or 1 = both
// (the single derived buffer of ABI revision 1)
inline bool flag_nib(int layouts) { return (layouts & 1) || (layouts & XFBQ_LAYOUT_NIBBLES); }
inline bool flag_tiles(int layouts) { return (layouts & 1) || (layouts & XFBQ_LAYOUT_TILES); }
}  // namespace

XFBQ_API int xfbq_scan_layouts(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k) {
    if (!width_ok(wd) || !width_ok(wq) || n < 1 || dim < 1 || nq < 1 || k < 1 || k > XFBQ_MAX_K) return 0;
    UmmaPlan up;
    if (make_umma_plan(n, dim, wd, nq, wq, k, true, &up) == XFBQ_OK && up.ok) return XFBQ_LAYOUT_TILES;
    CoopPlan cp;
    if (make_coop_plan(n, dim, wd, nq, wq, k, true, &cp) == XFBQ_OK && cp.ok) return XFBQ_LAYOUT_NIBBLES;
    MmaPlan mp;
    if (make_mma_plan(n, dim, wd, nq, wq, k, true, &mp) == XFBQ_OK && mp.ok) return XFBQ_LAYOUT_NIBBLES;
    return 0;
}

XFBQ_API int xfbq_kselect_small_f64(const void *db, const void *nib, int64_t n, int64_t dim, int wd, const double *queries, int64_t nq, int64_t ld,
                                    double scale, int wq, int k, int64_t extra_distance, int64_t row_offset, uint64_t *keys_out,
                                    uint64_t *cand_count_out, int64_t *cand_ids_out, int64_t cand_cap, int *inexact_out, uint64_t *nonfinite,
                                    void *workspace, int64_t workspace_bytes, void *stream) {
    if (!cand_count_out) return fail(XFBQ_E_INVALID, "null pointer");
    return search_small_impl(db, nib, n, dim, wd, queries, 1, nq, ld, scale, wq, k, row_offset, keys_out, nonfinite, workspace, workspace_bytes, stream,
                             extra_distance, cand_count_out, cand_ids_out, cand_cap, inexact_out);
}

XFBQ_API int64_t xfbq_scan_workspace_bytes(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k, int have_nibbles) {
    if (!width_ok(wd) || !width_ok(wq) || n < 0 || dim < 1 || nq < 0 || k < 1 || k > XFBQ_MAX_K) {
        fail(XFBQ_E_INVALID, "bad scan shape");
        return -1;
    }
    if (n == 0 || nq == 0) return 0;
    UmmaPlan up;
    if (make_umma_plan(n, dim, wd, nq, wq, k, flag_tiles(have_nibbles), &up)) return -1;
    if (up.ok) return static_cast<int64_t>(up.bytes);
    CoopPlan cp;
    if (make_coop_plan(n, dim, wd, nq, wq, k, flag_nib(have_nibbles), &cp)) return -1;
    if (cp.ok) return static_cast<int64_t>(cp.bytes);
    MmaPlan mp;
    if (make_mma_plan(n, dim, wd, nq, wq, k, flag_nib(have_nibbles), &mp, flag_tiles(have_nibbles))) return -1;
    if (mp.ok) return static_cast<int64_t>(mp.bytes);
    ScanPlan pl;
    if (make_plan(n, dim, wd, nq, wq, k, &pl)) return -1;
    if (pl.splits <= 1) return 0;
    return static_cast<int64_t>(pl.splits + merge_scratch_parts(pl.splits, k, nq)) * nq * k * 8;
}

XFBQ_API int xfbq_scan_plan(int64_t n, int64_t dim, int wd, int64_t nq, int wq, int k, int have_nibbles, int32_t out[6]) {
    if (!width_ok(wd) || !width_ok(wq) || n < 1 || dim < 1 || nq < 1 || k < 1 || k > XFBQ_MAX_K || !out)
        return fail(XFBQ_E_INVALID, "bad scan shape");
    UmmaPlan up;
    if (int rc = make_umma_plan(n, dim, wd, nq, wq, k, flag_tiles(have_nibbles), &up)) return rc;
    if (up.ok) {  // tcgen05 engine: tile = queries per CTA
        out[0] = 128 * up.main.MT; out[1] = up.main.groups; out[2] = up.main.parts; out[3] = up.main.cap;
        out[4] = 3; out[5] = static_cast<int32_t>(up.main.smem);
        return XFBQ_OK;
    }
    CoopPlan cp;
    if (int rc = make_coop_plan(n, dim, wd, nq, wq, k, flag_nib(have_nibbles), &cp)) return rc;
    if (cp.ok) {  // mma.sync engine, single-launch search: one 16-query tile, every warp of the grid keeps a list per query
        out[0] = 16; out[1] = 1; out[2] = cp.grid * coop::WARPS; out[3] = cp.cap;
        out[4] = 2; out[5] = static_cast<int32_t>(cp.smem);
        return XFBQ_OK;
    }
    MmaPlan mp;
    if (int rc = make_mma_plan(n, dim, wd, nq, wq, k, flag_nib(have_nibbles), &mp, flag_tiles(have_nibbles))) return rc;
    if (mp.ok) {  // integer-MMA engine: tile = queries per CTA
        out[0] = mp.main.QW * mp.main.QPW; out[1] = mp.main.groups; out[2] = mp.main.parts; out[3] = mp.main.cap;
        out[4] = 2; out[5] = static_cast<int32_t>(mp.main.smem);
        return XFBQ_OK;
    }
    ScanPlan pl;
    if (int rc = make_plan(n, dim, wd, nq, wq, k, &pl)) return rc;
    out[0] = pl.tq; out[1] = pl.q_tiles; out[2] = pl.splits; out[3] = pl.cap;
    out[4] = pl.fast ? 1 : 0; out[5] = static_cast<int32_t>(pl.smem);
    return XFBQ_OK;
}

XFBQ_API int xfbq_scan_topk(const void *db, const void *derived, int64_t n, int64_t dim, int wd, const uint32_t *q, int64_t nq,
                            int wq, int k, int64_t row_offset, uint64_t *keys_out, void *workspace,
                            int64_t workspace_bytes, void *stream) {
    // ABI revision 1: one derived buffer [nibble layout][byte tiles]
    const void *nib = nullptr, *tiles = nullptr;
    if (derived && n > 0 && dim >= 1 && width_ok(wd)) {
        if (nibble_region_bytes(n, dim, wd) > 0) nib = derived;
        if (tiles_supported(dim)) tiles = static_cast<const unsigned char *>(derived) + nibble_region_bytes(n, dim, wd);
    }
    return xfbq_scan_topk_layouts(db, nib, tiles, n, dim, wd, q, nq, wq, k, row_offset, keys_out, workspace, workspace_bytes, stream);
}

XFBQ_API int xfbq_scan_topk_layouts(const void *db, const void *nib, const void *tiles, int64_t n, int64_t dim, int wd, const uint32_t *q,
                                    int64_t nq, int wq, int k, int64_t row_offset, uint64_t *keys_out, void *workspace,
                                    int64_t workspace_bytes, void *stream) {
    if (!width_ok(wd) || !width_ok(wq)) return fail(XFBQ_E_INVALID, "bit width must be in 1..8, got %d/%d", wd, wq);
    if (n < 0 || dim < 1 || nq < 0) return fail(XFBQ_E_INVALID, "bad shape n=%lld dim=%lld nq=%lld", (long long)n, (long long)dim, (long long)nq);
    if (k < 1) return fail(XFBQ_E_INVALID, "k must be >= 1, got %d", k);
    if (k > XFBQ_MAX_K) return fail(XFBQ_E_UNSUPPORTED, "k=%d exceeds XFBQ_MAX_K=%d", k, XFBQ_MAX_K);
    if (row_offset < 0 || row_offset + n > (1ll << 32)) return fail(XFBQ_E_UNSUPPORTED, "row ids must fit 32 bits");
    if (xfbq_distance_upper_bound(dim, wd, wq) >= (1ll << 31)) return fail(XFBQ_E_UNSUPPORTED, "distance range exceeds 31 bits");
    if (nq == 0) return XFBQ_OK;
    if (!keys_out) return fail(XFBQ_E_INVALID, "null keys_out");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(keys_out, 0xFF, static_cast<size_t>(nq) * k * 8, st);
        if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "memset: %s", cudaGetErrorString(e));
        return XFBQ_OK;
    }
    if (!q) return fail(XFBQ_E_INVALID, "null pointer");
    UmmaPlan up;
    if (int rc = make_umma_plan(n, dim, wd, nq, wq, k, tiles != nullptr, &up)) return rc;
    if (up.ok) {
        if (!workspace || workspace_bytes < static_cast<int64_t>(up.bytes))
            return fail(XFBQ_E_INVALID, "workspace too small: need %zu bytes, got %lld", up.bytes, (long long)workspace_bytes);
        return run_umma(up, static_cast<unsigned char *>(workspace), tiles, n, dim, wd, q, nq, wq, k, row_offset, keys_out, st);
    }
    CoopPlan cp;
    if (int rc = make_coop_plan(n, dim, wd, nq, wq, k, nib != nullptr, &cp)) return rc;
    if (cp.ok) {
        if (!workspace || workspace_bytes < static_cast<int64_t>(cp.bytes))
            return fail(XFBQ_E_INVALID, "workspace too small: need %zu bytes, got %lld", cp.bytes, (long long)workspace_bytes);
        return run_coop(cp, static_cast<unsigned char *>(workspace), nib, n, dim, wd, q, nq, wq, k, row_offset, keys_out, st);
    }
    MmaPlan mp;
    if (int rc = make_mma_plan(n, dim, wd, nq, wq, k, nib != nullptr, &mp, tiles != nullptr)) return rc;
    if (mp.ok) {
        if (!workspace || workspace_bytes < static_cast<int64_t>(mp.bytes))
            return fail(XFBQ_E_INVALID, "workspace too small: need %zu bytes, got %lld", mp.bytes, (long long)workspace_bytes);
        const int C = static_cast<int>(chunks128(dim));
        unsigned char *ws = static_cast<unsigned char *>(workspace);
        uint32_t *qop = reinterpret_cast<uint32_t *>(ws + mp.off_qop);
        int32_t *qconst = reinterpret_cast<int32_t *>(ws + mp.off_qconst);
        mma::prep_queries_kernel<<<static_cast<unsigned>((mp.main.nq_pad * 32 + 255) / 256), 256, 0, st>>>(
            q, nq, mp.main.nq_pad, static_cast<int>(dim), wq, wd, C, qop, qconst);
        if (int rc = check_launch("prep_queries_kernel")) return rc;
        const int32_t *tau_init = nullptr;
        if (mp.sample && mp.count) {
            int32_t *tau = reinterpret_cast<int32_t *>(ws + mp.off_tau);
            if (int rc = run_counted_seed(ws, tiles, n, dim, wd, q, nq, wq, k, mp.sample,
                                          true, mp.off_uqimg, mp.off_uqconst, mp.off_seedpar, mp.off_seedhist, tau, st)) return rc;
            tau_init = tau;
        } else if (mp.sample) {
            uint64_t *prekeys = reinterpret_cast<uint64_t *>(ws + mp.off_prekeys);
            int32_t *tau = reinterpret_cast<int32_t *>(ws + mp.off_tau);
            if (int rc = run_mma_scan(mp.pre, mp, ws, nib, mp.sample, C, nq, k, row_offset, nullptr, prekeys, st)) return rc;
            mma::tau_from_keys_kernel<<<static_cast<unsigned>((nq + 255) / 256), 256, 0, st>>>(prekeys, qconst, nq, k, tau);
            if (int rc = check_launch("tau_from_keys_kernel")) return rc;
            tau_init = tau;
        }
        return run_mma_scan(mp.main, mp, ws, nib, n, C, nq, k, row_offset, tau_init, keys_out, st);
    }
    if (!db) return fail(XFBQ_E_INVALID, "this shape scans the bit planes (XOR/POPC kernels): the packed codes are required");
    ScanPlan pl;
    if (int rc = make_plan(n, dim, wd, nq, wq, k, &pl)) return rc;
    const int64_t need = pl.splits <= 1 ? 0 : static_cast<int64_t>(pl.splits + merge_scratch_parts(pl.splits, k, nq)) * nq * k * 8;
    if (need > 0 && (!workspace || workspace_bytes < need))
        return fail(XFBQ_E_INVALID, "workspace too small: need %lld bytes, got %lld", (long long)need, (long long)workspace_bytes);
    const int C = static_cast<int>(chunks128(dim));
    ScanKernel kern = pl.fast ? pick_kernel(wd, wq, C) : nullptr;
    if (!kern) kern = scan_topk_kernel<0, 0, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem));
    if (e != cudaSuccess) return fail(XFBQ_E_CUDA, "scan smem opt-in (%zu bytes): %s", pl.smem, cudaGetErrorString(e));
    ScanParams p;
    p.db = static_cast<const uint4 *>(db);
    p.n = n;
    p.row_offset = row_offset;
    p.q = q;
    p.out = pl.splits <= 1 ? keys_out : static_cast<uint64_t *>(workspace);
    p.nq = nq;
    p.split_steps = pl.split_steps;
    p.wd = wd; p.wq = wq; p.C = C;
    p.k = k; p.cap = pl.cap; p.tq = pl.tq;
    dim3 grid(static_cast<unsigned>(pl.splits), static_cast<unsigned>(pl.q_tiles));
    if (pl.q_tiles > 65535) return fail(XFBQ_E_UNSUPPORTED, "too many query tiles (%d); split the batch", pl.q_tiles);
    if (g_timing) timing_begin(st);
    kern<<<grid, SCAN_THREADS, pl.smem, st>>>(p);
    if (g_timing) timing_end(st);
    if (int rc = check_launch("scan_topk_kernel")) return rc;
    if (pl.splits > 1)
        return launch_merge(static_cast<const uint64_t *>(workspace), pl.splits, nq, k, keys_out,
                            static_cast<uint64_t *>(workspace) + static_cast<int64_t>(pl.splits) * nq * k, st);
    return XFBQ_OK;
}

XFBQ_API int xfbq_merge_topk(const uint64_t *keys_in, int parts, int64_t nq, int k, uint64_t *keys_out,
                             void *stream) {
    if (parts < 1 || nq < 0 || k < 1) return fail(XFBQ_E_INVALID, "bad merge shape parts=%d nq=%lld k=%d", parts, (long long)nq, k);
    if (k > XFBQ_MAX_K) return fail(XFBQ_E_UNSUPPORTED, "k=%d exceeds XFBQ_MAX_K=%d", k, XFBQ_MAX_K);
    if (nq == 0) return XFBQ_OK;
    if (!keys_in || !keys_out) return fail(XFBQ_E_INVALID, "null pointer");
    return launch_merge(keys_in, parts, nq, k, keys_out, nullptr, static_cast<cudaStream_t>(stream));
}

XFBQ_API int xfbq_unpack_keys(const uint64_t *keys, int64_t count, int64_t *dist, int64_t *ids, void *stream) {
    if (count < 0) return fail(XFBQ_E_INVALID, "negative count");
    if (count == 0) return XFBQ_OK;
    if (!keys || !dist || !ids) return fail(XFBQ_E_INVALID, "null pointer");
    unpack_keys_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(keys, count, dist, ids);
    return check_launch("unpack_keys_kernel");
}
