// Instruction-rate microbenchmark for the integer pipes the XFBQ scan can use on sm_100a.
// Measures lanes/clk/SM for POPC, LOP3, IADD3, IDP4A, IMAD, mixes, and legacy IMMA (int8 mma.sync).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

template <int OP>
__global__ void __launch_bounds__(512) k_alu(unsigned* out, unsigned seed, long long* clk) {
    unsigned v[CHAINS], acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) { v[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B9u; acc[c] = c; }
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (OP == 0) {            // POPC dependent chain
                v[c] = __popc(v[c]) + seed;  // popc + iadd
            } else if (OP == 1) {     // LOP3
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(acc[c]), "r"(seed));
            } else if (OP == 2) {     // IADD3
                asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(seed));
            } else if (OP == 3) {     // IDP4A
                asm volatile("dp4a.u32.s32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(v[c]), "r"(seed));
            } else if (OP == 4) {     // IMAD
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(seed), "r"(acc[c]));
            } else if (OP == 5) {     // POPC + 3 LOP3 (mix): does POPC overlap with ALU?
                unsigned p; asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(v[c]));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(p), "r"(seed));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(acc[c]) : "r"(v[c]), "r"(seed));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(acc[c]) : "r"(v[c]), "r"(seed));
            } else if (OP == 6) {     // pure POPC (no add), independent source mutated by lop3 every 4th
                unsigned p; asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(v[c]));
                acc[c] += p;
            } else if (OP == 7) {     // POPC + IDP4A mix
                unsigned p; asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(v[c]));
                asm volatile("dp4a.u32.s32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(p), "r"(seed));
            }
        }
    }
    long long t1 = clock64();
    unsigned r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= v[c] ^ acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// legacy int8 tensor path: mma.sync m16n8k32 u8 x s8 -> s32
__global__ void __launch_bounds__(512) k_imma(int* out, unsigned seed, long long* clk) {
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i + 1);
    for (int i = 0; i < 2; ++i) b[i] = seed * (threadIdx.x + i + 7);
    int c[CHAINS][4];
    for (int j = 0; j < CHAINS; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < CHAINS; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    long long t1 = clock64();
    int r = 0;
    for (int j = 0; j < CHAINS; ++j) for (int i = 0; i < 4; ++i) r ^= c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename F>
static void run(const char* name, F launch, int blocks, int threads, double ops_per_thread_iter, unsigned* out, long long* clk) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[4]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double cta_per_sm = (double)blocks / nsm;
    double lane_ops_cta = (double)threads * ITERS * CHAINS * ops_per_thread_iter;
    // per-SM rate from the in-kernel cycle count of CTA 0 (all CTAs of one SM run concurrently)
    double per_clk_sm = lane_ops_cta * cta_per_sm / (double)h[0];
    double total = lane_ops_cta * blocks;
    printf("{\"op\":\"%s\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"cycles_cta0\":%lld,\"lane_ops_per_clk_per_sm\":%.2f,\"G_lane_ops_per_s\":%.1f,\"eff_mhz\":%.0f}\n",
           name, blocks, threads, ms, h[0], per_clk_sm, total / ms / 1e6, (double)h[0] / ms / 1e3);
    cudaError_t err = cudaGetLastError(); if (err) printf("ERR %s\n", cudaGetErrorString(err));
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int threads = 512, per_sm = 2; int blocks = nsm * per_sm;
    unsigned* out; long long* clk;
    cudaMalloc(&out, (size_t)blocks * threads * 4); cudaMalloc(&clk, blocks * 8);
    printf("{\"sms\":%d}\n", nsm);
#define RUN(OP, NAME, OPS) run(NAME, [&] { k_alu<OP><<<blocks, threads>>>(out, 12345u, clk); }, blocks, threads, OPS, out, clk)
    RUN(0, "popc+iadd (count=1 popc)", 1);
    RUN(6, "popc+iadd indep (count=1 popc)", 1);
    RUN(1, "lop3", 1);
    RUN(2, "iadd", 1);
    RUN(3, "dp4a", 1);
    RUN(4, "imad", 1);
    RUN(5, "popc+3lop3 (count=4 ops)", 4);
    RUN(7, "popc+dp4a (count=2 ops)", 2);
    run("imma.16832 (count=1 mma per warp-lane)", [&] { k_imma<<<blocks, threads>>>((int*)out, 12345u, clk); }, blocks, threads, 1, out, clk);
    // for IMMA: lane_ops/clk/SM / 32 = warp-MMAs/clk/SM; x 16*8*32 MAC
    return 0;
}
