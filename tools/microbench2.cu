// IMMA.16832 latency / throughput vs independent chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
template <int CH>
__global__ void k(int* out, unsigned seed) {
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i + 1);
    for (int i = 0; i < 2; ++i) b[i] = seed * (threadIdx.x + i + 7);
    int c[CH][4];
    for (int j = 0; j < CH; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int r = 0;
    for (int j = 0; j < CH; ++j) for (int i = 0; i < 4; ++i) r ^= c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int CH>
void run(int warps_per_sm, int* out) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int threads = warps_per_sm * 32;
    for (int rep = 0; rep < 3; ++rep) k<CH><<<nsm, threads>>>(out, 12345u);
    cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int rep = 0; rep < 5; ++rep) k<CH><<<nsm, threads>>>(out, 12345u); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double mma_per_smsp = (double)warps_per_sm / 4.0 * ITERS * CH;     // per SMSP
    double clk = ms * 1e-3 * 1.965e9;
    printf("{\"chains\":%d,\"warps_per_sm\":%d,\"ms\":%.4f,\"clk_per_mma_per_smsp\":%.2f,\"chains_per_smsp\":%d,\"TMACs\":%.1f}\n",
           CH, warps_per_sm, ms, clk / mma_per_smsp, CH * warps_per_sm / 4, (double)nsm * warps_per_sm * ITERS * CH * 4096.0 / ms / 1e9);
}
int main() {
    int* out; cudaMalloc(&out, 148 * 1024 * 4);
    for (int w : {4, 8, 16, 32}) { run<1>(w, out); run<2>(w, out); run<4>(w, out); run<8>(w, out); run<16>(w, out); }
    return 0;
}
