// umma_probe.cu -- tcgen05 (UMMA) int8 bring-up and microbenchmarks for sm_100a.
//   test 1: correctness of one 128 x 256 x 256 s8 x s8 -> s32 tile (SWIZZLE_128B K-major smem operands,
//           descriptors built by hand) against a CPU GEMM
//   test 2: tcgen05.mma kind::i8 issue rate (MAC / clk / SM) for N = 256 and N = 128
//   test 3: tcgen05.ld throughput (B / clk / SM), 4 and 8 warps
//   test 4: both at once (does the accumulator drain slow the MMA pipe?)
// Every wait is bounded (clock64 time-out -> error flag), so a wrong descriptor cannot hang the GPU.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return done != 0;
}
__device__ __forceinline__ bool mbar_wait_bounded(uint64_t *bar, uint32_t parity, long long limit = 2000000000ll) {
    const long long t0 = clock64();
    while (!mbar_test(bar, parity))
        if (clock64() - t0 > limit) return false;
    return true;
}
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
// K-major SWIZZLE_128B operand descriptor: rows of 128 bytes, 8-row groups 1024 bytes apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);        // start address
    d |= static_cast<uint64_t>(1) << 16;                      // leading byte offset (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;              // stride byte offset: 8 rows x 128 B
    d |= static_cast<uint64_t>(1) << 46;                      // descriptor version (Blackwell)
    d |= static_cast<uint64_t>(2) << 61;                      // SWIZZLE_128B
    return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, bool a_signed, bool b_signed) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]),
          "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte offset of (row r, k byte kb) in a K-major SWIZZLE_128B operand of R rows and K = 128 * KB bytes
__host__ __device__ inline uint32_t sw128_offset(int r, int kbyte, int R) {
    const int blk = kbyte >> 7, kin = kbyte & 127;
    return static_cast<uint32_t>(blk * R * 128 + (r >> 3) * 1024 + (r & 7) * 128 + ((((kin >> 4) ^ (r & 7)) & 7) << 4) + (kin & 15));
}

constexpr int M_ = 128, N_ = 256, K_ = 256;

__device__ __forceinline__ void umma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- test 5: A operand in tensor memory
// Assumed layout: row m of A in lane m, column c holds K elements 4c..4c+3 (little endian), 8 columns per K = 32 step.
__global__ void __launch_bounds__(128, 1) tile_ts_kernel(const int8_t *A, const int8_t *B, int32_t *D, int *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sB = smem;       // 256 x 256 = 64 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < N_ * K_; i += blockDim.x) sB[sw128_offset(i / K_, i % K_, N_)] = static_cast<unsigned char>(B[i]);
    fence_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t a_tmem = tmem + 256;  // columns 256..319
    {
        const int m = warp * 32 + lane;
        const uint32_t *arow = reinterpret_cast<const uint32_t *>(A + m * K_);
        for (int c0 = 0; c0 < K_ / 4; c0 += 8) {
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = arow[c0 + j];
            tmem_st8(a_tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        }
        tmem_st_wait();
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = make_idesc(M_, N_, true, true);
        for (int ks = 0; ks < K_ / 32; ++ks) {
            const uint64_t bd = make_desc(smem_u32(sB) + (ks >> 2) * (N_ * 128) + (ks & 3) * 32);
            umma_i8_ts(tmem, a_tmem + ks * 8, bd, idesc, ks > 0 ? 1u : 0u);
        }
        umma_commit(&bar);
    }
    __syncwarp();
    if (!mbar_wait_bounded(&bar, 0)) { if (lane == 0) atomicExch(err, 1); }
    else {
        fence_after();
        for (int c0 = 0; c0 < N_; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N_ + c0 + j] = static_cast<int32_t>(v[j]);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- test 1
__global__ void __launch_bounds__(128, 1) tile_kernel(const int8_t *A, const int8_t *B, int32_t *D, int *err, int b_signed) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sA = smem;                 // 128 x 256 = 32 KB
    unsigned char *sB = smem + M_ * K_;       // 256 x 256 = 64 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < M_ * K_; i += blockDim.x) sA[sw128_offset(i / K_, i % K_, M_)] = static_cast<unsigned char>(A[i]);
    for (int i = threadIdx.x; i < N_ * K_; i += blockDim.x) sB[sw128_offset(i / K_, i % K_, N_)] = static_cast<unsigned char>(B[i]);
    fence_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 256);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    if (threadIdx.x == 0) {
        const uint32_t idesc = make_idesc(M_, N_, true, b_signed != 0);
        for (int ks = 0; ks < K_ / 32; ++ks) {
            const uint32_t koff = (ks >> 2) * 128 + 0;  // K block
            const uint64_t ad = make_desc(smem_u32(sA) + (ks >> 2) * (M_ * 128) + (ks & 3) * 32);
            const uint64_t bd = make_desc(smem_u32(sB) + (ks >> 2) * (N_ * 128) + (ks & 3) * 32);
            (void)koff;
            umma_i8(tmem, ad, bd, idesc, ks > 0 ? 1u : 0u);
        }
        umma_commit(&bar);
    }
    __syncwarp();
    if (!mbar_wait_bounded(&bar, 0)) { if (lane == 0) atomicExch(err, 1); }
    else {
        fence_after();
        for (int c0 = 0; c0 < N_; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N_ + c0 + j] = static_cast<int32_t>(v[j]);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------- tests 2-4
// warps 0..LW-1: tcgen05.ld loops (if do_ld); warp LW: MMA issuer (if do_mma).
template <int N, bool TS = false>
__global__ void __launch_bounds__(288, 1) rate_kernel(int iters_mma, int iters_ld, int do_mma, int do_ld, int ld_warps,
                                                      long long *mma_clk, long long *ld_clk, int *err, uint32_t *sink) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sA = smem;                 // 128 x 128 B
    unsigned char *sB = smem + 128 * 128;     // N x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 + N) * 128; i += blockDim.x) smem[i] = static_cast<unsigned char>((i * 2654435761u) >> 13) & 15;
    fence_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    if (warp == 8 && do_mma) {
        if (lane == 0) {
            const uint32_t idesc = make_idesc(128, N, true, true);
            const long long t0 = clock64();
            for (int it = 0; it < iters_mma; ++it) {
                const int ks = it & 3;
                const uint64_t ad = make_desc(smem_u32(sA) + ks * 32);
                const uint64_t bd = make_desc(smem_u32(sB) + ks * 32);
                if (TS) umma_i8_ts(tmem + ((it >> 2) & 1) * 128, tmem + 384 + ks * 8, bd, idesc, 1u);
                else umma_i8(tmem + ((it >> 2) & 1) * 256, ad, bd, idesc, 1u);
            }
            umma_commit(&bar);
            if (!mbar_wait_bounded(&bar, 0)) atomicExch(err, 2);
            mma_clk[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    } else if (warp < ld_warps && do_ld) {
        uint32_t acc = 0;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 256;
        const long long t0 = clock64();
        for (int it = 0; it < iters_ld; ++it) {
            uint32_t v[32];
            tmem_ld32(lane_base + (it & 7) * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= v[j];
        }
        const long long t1 = clock64();
        if (lane == 0) ld_clk[blockIdx.x * 8 + warp] = t1 - t0;
        if (acc == 0x12345678u) sink[0] = acc;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}


// ---------------------------------------------------------------- test 7: the scan kernel's issue pattern
// Groups of `gm` MMAs (M = 128, N = 128, K = 32, A in tensor memory) into `nacc` rotating 128-column accumulators.
// flags: 1 = tcgen05.commit after every group; 2 = the first MMA of a group overwrites (accumulate = 0);
// 4 = before issuing group g wait for the commit of group g - lag (an ideal, zero-work drain: the accumulator is free
// the moment its MMAs are done); 8 = a second warp waits for every commit and arrives on an "empty" barrier the issuer
// waits for instead (one hand-off hop, as in the real kernel with nothing to drain).
__global__ void __launch_bounds__(288, 1) pipe_kernel(int groups, int gm, int nacc, int lag, int flags, long long *clk, int *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sB = smem;  // 128 rows x 256 B (two K blocks)
    __shared__ uint64_t full[8], empty[8];
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 256; i += blockDim.x) smem[i] = static_cast<unsigned char>((i * 2654435761u) >> 13) & 15;
    fence_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t a_col = nacc * 128 <= 384 ? 384 : 0;  // four accumulators: the operand overlaps one (timing only)
    if (warp == 8) {
        if (lane == 0) {
            const uint32_t idesc = make_idesc(128, 128, true, (flags & 64) != 0);
            const uint64_t bd0 = make_desc(smem_u32(sB));
            const int bmask = (flags & 16) ? 0 : 1, amask = (flags & 32) ? 3 : 7;  // 16: one K block of B; 32: four column groups of A
            const uint32_t a0 = tmem + a_col;
            const bool first_overwrites = (flags & 2) != 0;
            const long long t0 = clock64();
            int buf = -1;
            for (int g = 0; g < groups; ++g) {
                buf = buf + 1 == nacc ? 0 : buf + 1;
                if ((flags & 4) && g >= lag) {
                    const int gw = g - lag;  // its commit went to full[gw % nacc], use number gw / nacc
                    if (flags & 8) { if (!mbar_wait_bounded(&empty[gw % nacc], (gw / nacc) & 1)) { atomicExch(err, 3); break; } }
                    else if (!mbar_wait_bounded(&full[gw % nacc], (gw / nacc) & 1)) { atomicExch(err, 3); break; }
                    fence_after();
                }
                const uint32_t d = tmem + buf * 128;
                for (int k0 = 0; k0 < gm; k0 += 8) {
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)
                        umma_i8_ts(d, a0 + (ks & amask) * 8, bd0 + ((((ks >> 2) & bmask) * (128 * 128) + (ks & 3) * 32) >> 4), idesc,
                                   (first_overwrites && k0 == 0 && ks == 0) ? 0u : 1u);
                }
                if (flags & 1) umma_commit(&full[buf]);
            }
            umma_commit(&full[7]);
            if (!mbar_wait_bounded(&full[7], 0)) atomicExch(err, 2);
            clk[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    } else if (warp == 0 && (flags & 8)) {
        for (int g = 0; g < groups; ++g) {  // the hop: every lane polls, lane 0 hands the accumulator back
            if (!mbar_wait_bounded(&full[g % nacc], (g / nacc) & 1)) { atomicExch(err, 4); break; }
            fence_after();
            fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[g % nacc])) : "memory");
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- test 8: the same with the scan kernel's issue idiom
// (whole warp walks the pipeline, one elected lane issues; 32-bit descriptor words, constant high word; waits with the
// retry loop inside the asm block).  flags as in test 7.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mbar_wait_tight(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
constexpr uint32_t P_DESC_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
template <bool ACC>
__device__ __forceinline__ void umma_i8_ts32(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\tsetp.ne.b32 p, %4, 0;\n\tmov.b64 db, {%2, %5};\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], db, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(idesc), "n"(ACC ? 1 : 0), "r"(P_DESC_HI) : "memory");
}
template <int GM, int NACC>
__global__ void __launch_bounds__(512, 1) pipe2_kernel(int groups, int lag, int flags, int hop_warps, long long *clk, int *err, int delay = 0) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sB = smem;  // 128 rows x 256 B (two K blocks)
    __shared__ uint64_t full[8], empty[8], bfull[4], bempty[4];
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 3 * 128 * 256; i += blockDim.x) smem[i] = static_cast<unsigned char>((i * 2654435761u) >> 13) & 15;
    fence_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) { mbar_init(&bfull[i], 1); mbar_init(&bempty[i], 1); }
        for (int i = 0; i < 8; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], hop_warps > 0 ? hop_warps : 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    constexpr uint32_t A_COL = NACC * 128 <= 384 ? 384 : 0;
    const uint32_t idesc = make_idesc(128, 128, true, false);
    if (warp == 12) {
        const uint32_t b_lo = ((smem_u32(sB) >> 4) & 0x3FFFu) | (1u << 16);
        const long long t0 = clock64();
        long long waited = 0;
        int buf = 0; uint32_t ph = 0;          // accumulator ring
        int wbuf = 0; uint32_t wph = 0;        // the group waited for (lag groups behind)
        int slot = 0; uint32_t sph = 0;        // operand ring (flags 512 / 1024): one slot per two groups
        for (int g = 0; g < groups; ++g) {
            if ((flags & 1024) && !(g & 1)) { mbar_wait_tight(&bfull[slot], sph); fence_after(); }
            if ((flags & 4) && g >= lag) {
                const long long w0 = clock64();
                mbar_wait_tight((flags & 8) ? &empty[wbuf] : &full[wbuf], wph);
                waited += clock64() - w0;
                fence_after();
                if (++wbuf == NACC) { wbuf = 0; wph ^= 1u; }
            }
            const uint32_t a_g = ((flags & 256) && (g & 1)) ? 64u : 0u;
            const uint32_t b_g = (flags & 1536) ? b_lo + static_cast<uint32_t>(slot) * ((128 * 256) >> 4) : b_lo;
            if (elect_one()) {
                const uint32_t d = tmem + buf * 128;
#pragma unroll
                for (int ks = 0; ks < GM; ++ks) {
                    const uint32_t ta = tmem + A_COL + a_g + (ks & 7) * 8;
                    const uint32_t bo = ((((ks >> 2) & 1) * (128 * 128)) + (ks & 3) * 32) >> 4;
                    if (ks == 0 && (flags & 2)) umma_i8_ts32<false>(d, ta, b_g + bo, idesc);
                    else umma_i8_ts32<true>(d, ta, b_g + bo, idesc);
                }
                if (flags & 1) umma_commit(&full[buf]);
            }
            __syncwarp();
            if (delay) {  // a dependent chain between two groups: is the issuer's path hidden behind queued MMAs?
                uint32_t x = static_cast<uint32_t>(g);
                for (int i = 0; i < delay; ++i) asm volatile("mad.lo.u32 %0, %0, 3, 1;" : "+r"(x));
                if (x == 0x7fffffffu) err[2] = 1;
            }
            if (++buf == NACC) { buf = 0; ph ^= 1u; }
            if ((flags & 1536) && (g & 1)) {
                if (flags & 1024) { if (elect_one()) umma_commit(&bempty[slot]); __syncwarp(); }
                if (++slot == 3) { slot = 0; sph ^= 1u; }
            }
        }
        if (elect_one()) umma_commit(&full[7]);
        __syncwarp();
        mbar_wait_tight(&full[7], 0);
        if (lane == 0) { clk[blockIdx.x] = clock64() - t0; clk[gridDim.x + blockIdx.x] = waited; }
        (void)ph;
    } else if (warp == 13 && (flags & 1024)) {
        if (lane == 0) {
            int slot = 0; uint32_t sph = 1;   // "empty" waits start on the completed phase
            for (int st = 0; st < groups / 2; ++st) {
                mbar_wait_tight(&bempty[slot], sph);
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bfull[slot])) : "memory");
                if (++slot == 3) { slot = 0; sph ^= 1u; }
            }
        }
        __syncwarp();
    } else if (warp < hop_warps && (flags & 8)) {
        int buf = 0; uint32_t ph = 0;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        uint32_t sinkv = 0;
        for (int g = 0; g < groups; ++g) {  // the hop: every lane polls, [reads its share of the accumulator], lane 0 hands it back
            mbar_wait_tight(&full[buf], ph);
            fence_after();
            if (flags & 128) {
                uint32_t v[32];
                tmem_ld32(lane_base + buf * 128 + ((warp >> 2) & 1) * 64, v);
                tmem_ld32(lane_base + buf * 128 + ((warp >> 2) & 1) * 64 + 32, v);
                tmem_ld_wait();
                sinkv ^= v[0];
            }
            fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[buf])) : "memory");
            if (++buf == NACC) { buf = 0; ph ^= 1u; }
        }
        if (sinkv == 0x12345u) err[1] = 1;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- test 9: how far ahead of the tensor pipe can the issuer run?
// From an idle pipe, one elected lane issues K MMAs (128 x 128 x 32, A in tensor memory) back to back and reads the clock after the
// last one was ACCEPTED (not completed): the time stays flat up to the depth of the instruction queue, then grows by one MMA time each.
template <int K>
__global__ void __launch_bounds__(128, 1) queue_kernel(long long *clk, int *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 256; i += blockDim.x) smem[i] = static_cast<unsigned char>((i * 2654435761u) >> 13) & 15;
    fence_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t idesc = make_idesc(128, 128, true, false);
    if (warp == 1) {
        const uint32_t b_lo = ((smem_u32(smem) >> 4) & 0x3FFFu) | (1u << 16);
        long long best_issue = 1ll << 60, best_total = 0;
        for (int rep = 0; rep < 8; ++rep) {
            long long t0 = 0, t1 = 0;
            if (elect_one()) {
                t0 = clock64();
#pragma unroll
                for (int ks = 0; ks < K; ++ks)
                    umma_i8_ts32<true>(tmem + (ks >> 3) * 128, tmem + 384 + (ks & 7) * 8, b_lo + (((((ks >> 2) & 1) * (128 * 128)) + (ks & 3) * 32) >> 4), idesc);
                t1 = clock64();
                umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait_tight(&bar, rep & 1);
            const long long t2 = clock64();
            t0 = __shfl_sync(0xffffffffu, t0, __ffs(__ballot_sync(0xffffffffu, t0 != 0)) - 1);
            t1 = __shfl_sync(0xffffffffu, t1, __ffs(__ballot_sync(0xffffffffu, t1 != 0)) - 1);
            if (t1 - t0 < best_issue) { best_issue = t1 - t0; best_total = t2 - t0; }
        }
        if (lane == 0) { clk[blockIdx.x * 2] = best_issue; clk[blockIdx.x * 2 + 1] = best_total; }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
    (void)err;
}

// ---------------------------------------------------------------- test 11: do queued MMAs execute while the issuing warp computes?
// Warp 1 issues 8 MMAs + commit, then runs a dependent integer chain of `delay` iterations and reads the clock; warp 2 polls the
// commit barrier and reads the clock when the MMAs are done.  Both relative to the same start (a CTA barrier).
__global__ void __launch_bounds__(128, 1) overlap_kernel(int delay, long long *clk, int *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 256; i += blockDim.x) smem[i] = static_cast<unsigned char>((i * 2654435761u) >> 13) & 15;
    fence_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t idesc = make_idesc(128, 128, true, false);
    for (int rep = 0; rep < 4; ++rep) {
        __syncthreads();
        const long long t0 = clock64();
        if (warp == 1) {
            const uint32_t b_lo = ((smem_u32(smem) >> 4) & 0x3FFFu) | (1u << 16);
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_i8_ts32<true>(tmem, tmem + 384 + (ks & 7) * 8, b_lo + (((((ks >> 2) & 1) * (128 * 128)) + (ks & 3) * 32) >> 4), idesc);
                umma_commit(&bar);
            }
            __syncwarp();
            const long long t1 = clock64();
            uint32_t x = static_cast<uint32_t>(rep);
            for (int i = 0; i < delay; ++i) asm volatile("mad.lo.u32 %0, %0, 3, 1;" : "+r"(x));
            const long long t2 = clock64();
            if (x == 0x7fffffffu) err[2] = 1;
            if (lane == 0) { clk[0] = t1 - t0; clk[1] = t2 - t0; }
        } else if (warp == 2) {
            mbar_wait_tight(&bar, rep & 1);
            const long long t3 = clock64();
            if (lane == 0) clk[2] = t3 - t0;
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- test 12: two issuing warps, alternate groups
// Warps 12 and 13 issue the even / odd groups (8 MMAs + commit each) into rotating accumulators; before group g a warp waits
// for the commit of group g - 2 (flags & 4) -- and, to keep the two streams in step, for nothing else.  A dependent chain of
// `delay` iterations follows every group, as in test 10: with one warp it is fully exposed, with two it should hide.
template <int NACC>
__global__ void __launch_bounds__(512, 1) pipe3_kernel(int groups, int flags, int delay, int issuers, long long *clk, int *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t full[8];
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 256; i += blockDim.x) smem[i] = static_cast<unsigned char>((i * 2654435761u) >> 13) & 15;
    fence_async_smem();
    if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t idesc = make_idesc(128, 128, true, false);
    if (warp >= 12 && warp < 12 + issuers) {
        const int me = warp - 12;
        const uint32_t b_lo = ((smem_u32(smem) >> 4) & 0x3FFFu) | (1u << 16);
        const long long t0 = clock64();
        for (int g = me; g < groups; g += issuers) {
            const int buf = g % NACC;
            if ((flags & 4) && g >= 2) { const int gw = g - 2; mbar_wait_tight(&full[gw % NACC], (gw / NACC) & 1); fence_after(); }
            if (elect_one()) {
                const uint32_t d = tmem + buf * 128;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint32_t bo = ((((ks >> 2) & 1) * (128 * 128)) + (ks & 3) * 32) >> 4;
                    if (ks == 0) umma_i8_ts32<false>(d, tmem + 384 + (g & 1) * 64 + ks * 8, b_lo + bo, idesc);
                    else umma_i8_ts32<true>(d, tmem + 384 + (g & 1) * 64 + ks * 8, b_lo + bo, idesc);
                }
                umma_commit(&full[buf]);
            }
            __syncwarp();
            if (delay) {
                uint32_t x = static_cast<uint32_t>(g);
                for (int i = 0; i < delay; ++i) asm volatile("mad.lo.u32 %0, %0, 3, 1;" : "+r"(x));
                if (x == 0x7fffffffu) err[2] = 1;
            }
        }
        if (elect_one()) umma_commit(&full[6 + me]);
        __syncwarp();
        mbar_wait_tight(&full[6 + me], 0);
        if (lane == 0) clk[blockIdx.x * 2 + me] = clock64() - t0;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- test 13: are two concurrently issued MMA chains independent?
// Warps 1 and 2 each issue 8 MMAs (K = 256) of their own query tile (A0 / A1 in tensor memory) against the same documents into
// their own accumulator, at the same time (mode 0) or one after the other (mode 1); both accumulators are checked against the CPU.
__global__ void __launch_bounds__(128, 1) two_chain_kernel(const int8_t *A, const int8_t *B, int32_t *D, int mode, int *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sB = smem;       // 128 x 256
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 256; i += blockDim.x) sB[sw128_offset(i / 256, i % 256, 128)] = static_cast<unsigned char>(B[i]);
    fence_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc(&tmem_base_s, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_s;
    {
        const int m = warp * 32 + lane;
        for (int tile = 0; tile < 2; ++tile) {
            const uint32_t *arow = reinterpret_cast<const uint32_t *>(A + (tile * 128 + m) * 256);
            for (int c0 = 0; c0 < 64; c0 += 8) {
                uint32_t v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = arow[c0 + j];
                tmem_st8(tmem + 256 + tile * 64 + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            }
        }
        tmem_st_wait();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t idesc = make_idesc(128, 128, true, false);
    for (int rep = 0; rep < 64; ++rep) {
        __syncthreads();
        if (warp == 1 || warp == 2) {
            const int me = warp - 1;
            if (mode == 1 && me == 1) { mbar_wait_tight(&bar[0], rep & 1); fence_after(); }
            const uint32_t b_lo = ((smem_u32(sB) >> 4) & 0x3FFFu) | (1u << 16);
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint32_t bo = ((((ks >> 2) & 1) * (128 * 128)) + (ks & 3) * 32) >> 4;
                    if (ks == 0) umma_i8_ts32<false>(tmem + me * 128, tmem + 256 + me * 64 + ks * 8, b_lo + bo, idesc);
                    else umma_i8_ts32<true>(tmem + me * 128, tmem + 256 + me * 64 + ks * 8, b_lo + bo, idesc);
                }
                umma_commit(&bar[me]);
            }
            __syncwarp();
        }
        mbar_wait_tight(&bar[0], rep & 1);
        mbar_wait_tight(&bar[1], rep & 1);
        fence_after();
        // check against the first repetition's result (kept in registers), report differences
        for (int acc = 0; acc < 2; ++acc)
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + acc * 128 + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    int32_t *dst = D + ((acc * 128 + warp * 32 + lane) * 128 + c0 + j);
                    if (rep == 0) *dst = static_cast<int32_t>(v[j]);
                    else if (*dst != static_cast<int32_t>(v[j])) atomicAdd(err + 1, 1);
                }
            }
        fence_before();
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main(int argc, char **argv) {
    int which = argc > 1 ? atoi(argv[1]) : 0;
    int *err;
    CK(cudaMalloc(&err, 4));
    CK(cudaMemset(err, 0, 4));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    if (which == 0 || which == 1) {
        for (int b_signed = 1; b_signed >= 0; --b_signed) {
            std::vector<int8_t> A(M_ * K_), B(N_ * K_);
            srand(1234);
            for (auto &a : A) a = static_cast<int8_t>(2 * (rand() % 16) - 15);
            for (auto &b : B) b = static_cast<int8_t>(rand() % 16);
            int8_t *dA, *dB; int32_t *dD;
            CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, M_ * N_ * 4));
            CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
            CK(cudaMemset(dD, 0xCC, M_ * N_ * 4));
            const int smem = M_ * K_ + N_ * K_;
            CK(cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            tile_kernel<<<1, 128, smem>>>(dA, dB, dD, err, b_signed);
            CK(cudaDeviceSynchronize());
            int herr = 0;
            CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
            std::vector<int32_t> D(M_ * N_);
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            long long bad = 0; int first = -1;
            for (int m = 0; m < M_; ++m)
                for (int n = 0; n < N_; ++n) {
                    int32_t s = 0;
                    for (int k = 0; k < K_; ++k) s += static_cast<int32_t>(A[m * K_ + k]) * static_cast<int32_t>(B[n * K_ + k]);
                    if (s != D[m * N_ + n]) { if (first < 0) first = m * N_ + n; ++bad; }
                }
            printf("{\"test\": \"tile_128x256x256_i8\", \"b_signed\": %d, \"timeout\": %d, \"mismatches\": %lld, \"first_bad\": %d, \"d0\": %d}\n",
                   b_signed, herr, bad, first, D[0]);
            fflush(stdout);
            CK(cudaMemset(err, 0, 4));
        }
    }
    if (which == 0 || which == 5) {
        std::vector<int8_t> A(M_ * K_), B(N_ * K_);
        srand(4321);
        for (auto &a : A) a = static_cast<int8_t>(2 * (rand() % 16) - 15);
        for (auto &b : B) b = static_cast<int8_t>(rand() % 16);
        int8_t *dA, *dB; int32_t *dD;
        CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, M_ * N_ * 4));
        CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
        CK(cudaMemset(dD, 0xCC, M_ * N_ * 4));
        const int smem = N_ * K_;
        CK(cudaFuncSetAttribute(tile_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        tile_ts_kernel<<<1, 128, smem>>>(dA, dB, dD, err);
        CK(cudaDeviceSynchronize());
        int herr = 0;
        CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
        std::vector<int32_t> D(M_ * N_);
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        long long bad = 0; int first = -1;
        for (int m = 0; m < M_; ++m)
            for (int n = 0; n < N_; ++n) {
                int32_t s = 0;
                for (int k = 0; k < K_; ++k) s += static_cast<int32_t>(A[m * K_ + k]) * static_cast<int32_t>(B[n * K_ + k]);
                if (s != D[m * N_ + n]) { if (first < 0) first = m * N_ + n; ++bad; }
            }
        printf("{\"test\": \"tile_ts_128x256x256_i8 (A in TMEM)\", \"timeout\": %d, \"mismatches\": %lld, \"first_bad\": %d, \"d0\": %d}\n", herr, bad, first, D[0]);
        fflush(stdout);
        CK(cudaMemset(err, 0, 4));
    }
    long long *mma_clk, *ld_clk; uint32_t *sink;
    CK(cudaMalloc(&mma_clk, sms * 8)); CK(cudaMalloc(&ld_clk, sms * 64)); CK(cudaMalloc(&sink, 4));
    auto run_rate = [&](int N, int do_mma, int do_ld, int ld_warps, bool ts = false) -> int {
        const int iters_mma = 8192, iters_ld = 4096;
        const int smem = (128 + N) * 128;
        CK(cudaMemset(mma_clk, 0, sms * 8)); CK(cudaMemset(ld_clk, 0, sms * 64));
        if (N == 256) {
            CK(cudaFuncSetAttribute(rate_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            rate_kernel<256><<<sms, 288, smem>>>(iters_mma, iters_ld, do_mma, do_ld, ld_warps, mma_clk, ld_clk, err, sink);
        } else if (ts) {
            CK(cudaFuncSetAttribute(rate_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            rate_kernel<128, true><<<sms, 288, smem>>>(iters_mma, iters_ld, do_mma, do_ld, ld_warps, mma_clk, ld_clk, err, sink);
        } else {
            CK(cudaFuncSetAttribute(rate_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            rate_kernel<128><<<sms, 288, smem>>>(iters_mma, iters_ld, do_mma, do_ld, ld_warps, mma_clk, ld_clk, err, sink);
        }
        CK(cudaDeviceSynchronize());
        int herr = 0;
        CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
        std::vector<long long> mc(sms), lc(sms * 8);
        CK(cudaMemcpy(mc.data(), mma_clk, sms * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(lc.data(), ld_clk, sms * 64, cudaMemcpyDeviceToHost));
        long long mmax = 0, lmax = 0;
        for (auto v : mc) if (v > mmax) mmax = v;
        for (auto v : lc) if (v > lmax) lmax = v;
        const double mac_per_clk = do_mma && mmax ? 128.0 * N * 32 * iters_mma / mmax : 0.0;
        const double ld_bytes_per_clk = do_ld && lmax ? 4096.0 * iters_ld * ld_warps / lmax : 0.0;
        printf("{\"test\": \"rate%s\", \"N\": %d, \"mma\": %d, \"ld\": %d, \"ld_warps\": %d, \"timeout\": %d, \"mma_clk_per_inst\": %.1f, "
               "\"mac_per_clk_per_sm\": %.0f, \"ld_clk_per_inst\": %.1f, \"ld_bytes_per_clk_per_sm\": %.1f}\n",
               ts ? "_ts" : "", N, do_mma, do_ld, ld_warps, herr, do_mma ? double(mmax) / iters_mma : 0.0, mac_per_clk,
               do_ld ? double(lmax) / iters_ld : 0.0, ld_bytes_per_clk);
        fflush(stdout);
        CK(cudaMemset(err, 0, 4));
        return 0;
    };
    if (which == 0 || which == 2) { if (run_rate(256, 1, 0, 0)) return 1; if (run_rate(128, 1, 0, 0)) return 1; }
    if (which == 0 || which == 3) { if (run_rate(256, 0, 1, 4)) return 1; if (run_rate(256, 0, 1, 8)) return 1; }
    if (which == 0 || which == 4) { if (run_rate(256, 1, 1, 4)) return 1; if (run_rate(256, 1, 1, 8)) return 1; if (run_rate(128, 1, 1, 8)) return 1; }
    if (which == 0 || which == 6) { if (run_rate(128, 1, 0, 0, true)) return 1; if (run_rate(128, 1, 1, 8, true)) return 1; }
    if (which == 0 || which == 7) {
        const int smem = 128 * 256;
        CK(cudaFuncSetAttribute(pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        struct Cfg { int gm, nacc, lag, flags; };
        const Cfg cfgs[] = {{8, 3, 0, 16}, {8, 3, 0, 32}, {8, 3, 0, 64}, {8, 3, 0, 112}, {8, 2, 0, 112}, {8, 1, 0, 112}, {8, 1, 0, 0}, {8, 3, 0, 0}, {8, 3, 0, 1}, {8, 3, 0, 2}, {8, 3, 0, 3}, {8, 3, 2, 7}, {8, 3, 1, 7}, {8, 3, 2, 15}, {8, 4, 3, 7}, {8, 4, 3, 15},
                            {16, 3, 2, 7}, {16, 3, 2, 15}, {8, 2, 1, 7}, {8, 2, 1, 15}};
        for (const Cfg &c : cfgs) {
            const int groups = 4096;
            CK(cudaMemset(mma_clk, 0, sms * 8));
            pipe_kernel<<<sms, 288, smem>>>(groups, c.gm, c.nacc, c.lag, c.flags, mma_clk, err);
            CK(cudaDeviceSynchronize());
            int herr = 0;
            CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
            std::vector<long long> mc(sms);
            CK(cudaMemcpy(mc.data(), mma_clk, sms * 8, cudaMemcpyDeviceToHost));
            long long mmax = 0;
            for (auto v : mc) if (v > mmax) mmax = v;
            printf("{\"test\": \"pipe\", \"mmas_per_group\": %d, \"accumulators\": %d, \"lag\": %d, \"flags\": %d, \"timeout\": %d, "
                   "\"clk_per_group\": %.1f, \"clk_per_mma\": %.2f}\n", c.gm, c.nacc, c.lag, c.flags, herr, double(mmax) / groups, double(mmax) / groups / c.gm);
            fflush(stdout);
            CK(cudaMemset(err, 0, 4));
        }
    }
    if (which == 0 || which == 8) {
        const int smem = 3 * 128 * 256;
        struct Cfg { int gm, nacc, lag, flags, hop; };
        const Cfg cfgs[] = {{8, 3, 0, 3, 0}, {8, 3, 2, 7, 0}, {8, 3, 2, 143, 8}, {8, 3, 2, 143 + 256, 8}, {8, 3, 2, 143 + 512, 8}, {8, 3, 2, 143 + 768, 8}, {8, 3, 2, 143 + 1024, 8}, {8, 3, 2, 143 + 1024 + 256, 8}, {8, 3, 3, 143 + 1024 + 256, 8}, {8, 3, 1, 143, 8},
                            {8, 4, 3, 7, 0}, {8, 4, 3, 15, 8}, {8, 4, 2, 15, 8}, {16, 3, 2, 7, 0}, {16, 3, 2, 15, 8}, {16, 3, 2, 143, 8}, {8, 2, 1, 7, 0}, {8, 2, 1, 15, 8}};
        for (const Cfg &c : cfgs) {
            const int groups = 4096;
            CK(cudaMemset(mma_clk, 0, sms * 8));
            long long *clk2; CK(cudaMalloc(&clk2, sms * 16)); CK(cudaMemset(clk2, 0, sms * 16));
#define RUN_PIPE2(GM, NACC) do { CK(cudaFuncSetAttribute(pipe2_kernel<GM, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
            pipe2_kernel<GM, NACC><<<sms, 512, smem>>>(groups, c.lag, c.flags, c.hop, clk2, err); } while (0)
            if (c.gm == 8 && c.nacc == 3) RUN_PIPE2(8, 3); else if (c.gm == 8 && c.nacc == 4) RUN_PIPE2(8, 4);
            else if (c.gm == 8 && c.nacc == 2) RUN_PIPE2(8, 2); else RUN_PIPE2(16, 3);
            CK(cudaDeviceSynchronize());
            int herr = 0;
            CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
            std::vector<long long> mc(2 * sms);
            CK(cudaMemcpy(mc.data(), clk2, sms * 16, cudaMemcpyDeviceToHost));
            CK(cudaFree(clk2));
            long long mmax = 0, wmax = 0;
            for (int i = 0; i < sms; ++i) { if (mc[i] > mmax) mmax = mc[i]; if (mc[sms + i] > wmax) wmax = mc[sms + i]; }
            printf("{\"test\": \"pipe2\", \"mmas_per_group\": %d, \"accumulators\": %d, \"lag\": %d, \"flags\": %d, \"hop_warps\": %d, \"timeout\": %d, "
                   "\"clk_per_group\": %.1f, \"clk_per_mma\": %.2f, \"issuer_wait_clk_per_group\": %.1f}\n", c.gm, c.nacc, c.lag, c.flags, c.hop, herr,
                   double(mmax) / groups, double(mmax) / groups / c.gm, double(wmax) / groups);
            fflush(stdout);
            CK(cudaMemset(err, 0, 4));
        }
    }
    if (which == 0 || which == 9) {
        const int smem = 128 * 256;
        long long *clk2; CK(cudaMalloc(&clk2, 16)); 
        long long h[2];
#define RUN_Q(K) do { CK(cudaFuncSetAttribute(queue_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); CK(cudaMemset(clk2, 0, 16)); \
        queue_kernel<K><<<1, 128, smem>>>(clk2, err); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, clk2, 16, cudaMemcpyDeviceToHost)); \
        printf("{\"test\": \"issue_queue\", \"mmas\": %d, \"clk_until_last_accepted\": %lld, \"clk_until_complete\": %lld}\n", K, h[0], h[1]); fflush(stdout); } while (0)
        RUN_Q(1); RUN_Q(2); RUN_Q(3); RUN_Q(4); RUN_Q(5); RUN_Q(6); RUN_Q(8); RUN_Q(10); RUN_Q(12); RUN_Q(16); RUN_Q(24);
        CK(cudaFree(clk2));
    }
    if (which == 10) {
        const int smem = 3 * 128 * 256;
        const int groups = 4096;
        long long *clk2; CK(cudaMalloc(&clk2, sms * 16));
        CK(cudaFuncSetAttribute(pipe2_kernel<8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int flags : {0, 2, 1, 3, 143}) for (int delay : {0, 4, 32, 128}) {
            CK(cudaMemset(clk2, 0, sms * 16));
            pipe2_kernel<8, 3><<<sms, 512, smem>>>(groups, 2, flags, 8, clk2, err, delay);
            CK(cudaDeviceSynchronize());
            std::vector<long long> mc(2 * sms);
            CK(cudaMemcpy(mc.data(), clk2, sms * 16, cudaMemcpyDeviceToHost));
            long long mmax = 0;
            for (int i = 0; i < sms; ++i) if (mc[i] > mmax) mmax = mc[i];
            printf("{\"test\": \"pipe2_delay\", \"flags\": %d, \"delay_iters\": %d, \"clk_per_group\": %.1f}\n", flags, delay, double(mmax) / groups);
            fflush(stdout);
        }
        CK(cudaFree(clk2));
    }
    if (which == 11) {
        const int smem = 128 * 256;
        long long *clk2; CK(cudaMalloc(&clk2, 32));
        long long h[3];
        CK(cudaFuncSetAttribute(overlap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int delay : {0, 32, 128, 512}) {
            CK(cudaMemset(clk2, 0, 32));
            overlap_kernel<<<1, 128, smem>>>(delay, clk2, err);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, clk2, 24, cudaMemcpyDeviceToHost));
            printf("{\"test\": \"overlap\", \"delay_iters\": %d, \"issued_at\": %lld, \"issuer_chain_done_at\": %lld, \"mmas_complete_at\": %lld}\n", delay, h[0], h[1], h[2]);
            fflush(stdout);
        }
        CK(cudaFree(clk2));
    }
    if (which == 12) {
        const int smem = 128 * 256;
        const int groups = 4096;
        long long *clk2; CK(cudaMalloc(&clk2, sms * 16));
        CK(cudaFuncSetAttribute(pipe3_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int issuers : {1, 2}) for (int flags : {0, 4}) for (int delay : {0, 4, 32, 64, 128}) {
            CK(cudaMemset(clk2, 0, sms * 16));
            pipe3_kernel<3><<<sms, 512, smem>>>(groups, flags, delay, issuers, clk2, err);
            CK(cudaDeviceSynchronize());
            std::vector<long long> mc(2 * sms);
            CK(cudaMemcpy(mc.data(), clk2, sms * 16, cudaMemcpyDeviceToHost));
            long long mmax = 0;
            for (int i = 0; i < 2 * sms; ++i) if (mc[i] > mmax) mmax = mc[i];
            int herr = 0; CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
            printf("{\"test\": \"pipe3\", \"issuers\": %d, \"flags\": %d, \"delay_iters\": %d, \"err\": %d, \"clk_per_group\": %.1f}\n", issuers, flags, delay, herr, double(mmax) / groups);
            fflush(stdout);
        }
        CK(cudaFree(clk2));
    }
    if (which == 13) {
        std::vector<int8_t> A(256 * 256), B(128 * 256);
        srand(777);
        for (auto &a : A) a = static_cast<int8_t>(2 * (rand() % 16) - 15);
        for (auto &b : B) b = static_cast<int8_t>(rand() % 16);
        int8_t *dA, *dB; int32_t *dD; int *err2;
        CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, 256 * 128 * 4)); CK(cudaMalloc(&err2, 16));
        CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
        const int smem = 128 * 256;
        CK(cudaFuncSetAttribute(two_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int mode = 0; mode < 2; ++mode) {
            CK(cudaMemset(dD, 0xCC, 256 * 128 * 4)); CK(cudaMemset(err2, 0, 16));
            two_chain_kernel<<<1, 128, smem>>>(dA, dB, dD, mode, err2);
            CK(cudaDeviceSynchronize());
            int herr[4];
            CK(cudaMemcpy(herr, err2, 16, cudaMemcpyDeviceToHost));
            std::vector<int32_t> D(256 * 128);
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            long long bad = 0;
            for (int m = 0; m < 256; ++m)
                for (int n = 0; n < 128; ++n) {
                    int32_t acc = 0;
                    for (int k = 0; k < 256; ++k) acc += static_cast<int32_t>(A[m * 256 + k]) * static_cast<int32_t>(static_cast<uint8_t>(B[n * 256 + k]));
                    if (acc != D[m * 128 + n]) ++bad;
                }
            printf("{\"test\": \"two_chains\", \"mode\": \"%s\", \"mismatches_vs_cpu_first_rep\": %lld, \"changes_in_later_reps\": %d}\n",
                   mode ? "one after the other" : "concurrent", bad, herr[1]);
            fflush(stdout);
        }
    }
    return 0;
}
