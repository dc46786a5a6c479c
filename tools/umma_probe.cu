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
    return 0;
}
