// Which hand-off / barrier forms do compute-sanitizer's racecheck and synccheck accept?  (tools/, not product code)
// Producer warp 0 writes a shared row and signals; consumer warp 1 polls, reads the row, releases the slot.
// variant 0: mbarrier.arrive / mbarrier.test_wait poll      1: arrive / try_wait loop
// variant 2: like 1 + roles meet at `bar.sync 0` from two call sites     3: roles meet at `bar.sync 1, 64`
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory"); }
__device__ __forceinline__ bool mb_test(uint64_t *b, uint32_t ph) {
    uint32_t d; asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(s32(b)), "r"(ph) : "memory"); return d; }
__device__ __forceinline__ bool mb_try(uint64_t *b, uint32_t ph) {
    uint32_t d; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(s32(b)), "r"(ph) : "memory"); return d; }
// variant 4: the queue kernel's shape -- 32 slots, lane l of the producer warp fills slot l and arrives on ITS mbarrier,
// lane l of the consumer warp tests ITS mbarrier (32 different barrier addresses in one warp instruction), reads, releases
__global__ void probe_lanes(int rounds, int *out) {
    __shared__ int rows[32][4];
    __shared__ uint64_t full[32], empty[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 32) { mb_init(&full[lane], 1); mb_init(&empty[lane], 1); }
    __syncthreads();
    int acc = 0;
    if (warp == 0) {
        for (int r = 0; r < rounds; ++r) {
            while (!mb_test(&empty[lane], (r & 1) ^ 1)) {}
            for (int i = 0; i < 4; ++i) rows[lane][i] = r * 4 + i + lane;
            mb_arrive(&full[lane]);
            __syncwarp();
        }
    } else {
        for (int r = 0; r < rounds; ++r) {
            bool done = false;
            while (!__all_sync(0xffffffffu, done)) {   // poll like the resolver: test, vote, consume what is ready
                const bool ready = !done && mb_test(&full[lane], r & 1);
                const unsigned m = __ballot_sync(0xffffffffu, ready);
                if (m == 0) continue;
                if (ready) {
                    for (int i = 0; i < 4; ++i) acc += rows[lane][i];
                    mb_arrive(&empty[lane]);
                    done = true;
                }
                __syncwarp();
            }
        }
        atomicAdd(out, acc);
    }
}
// variant 5: one 64-slot ring with running tickets, a varying number of rows parked per round (lanes < n_r), the consumer
// lane i takes ticket tail + i: every lane meets every slot's barrier over time, exactly the queue kernel's protocol
__global__ void probe_ring(int rounds, int *out) {
    constexpr int R = 64, LOG_R = 6;
    __shared__ int rows[R][4];
    __shared__ uint64_t full[R], empty[R], done_bar;
    __shared__ int fin;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < R; i += blockDim.x) { mb_init(&full[i], 1); mb_init(&empty[i], 1); }
    if (threadIdx.x == 0) mb_init(&done_bar, 1);
    __syncthreads();
    if (warp == 0) {
        int head = 0;
        for (int r = 0; r < rounds; ++r) {
            const int n = 1 + (r * 7) % 32;
            if (lane < n) {
                const int t = head + lane, slot = t & (R - 1);
                const uint32_t par = ((t >> LOG_R) & 1) ^ 1;
                while (!mb_test(&empty[slot], par)) {}
                for (int i = 0; i < 4; ++i) rows[slot][i] = t + i;
                mb_arrive(&full[slot]);
            }
            head += n;
            __syncwarp();
        }
        if (lane == 0) { fin = head; mb_arrive(&done_bar); }
    } else {
        int tail = 0, acc = 0;
        while (true) {
            const int t = tail + lane, slot = t & (R - 1);
            const bool ready = mb_test(&full[slot], (t >> LOG_R) & 1);
            const unsigned rm = __ballot_sync(0xffffffffu, ready);
            const int n = rm == 0xffffffffu ? 32 : __ffs(~rm) - 1;
            if (n == 0) {
                if (mb_test(&done_bar, 0) && fin == tail) break;
                continue;
            }
            if (lane < n) {
                for (int i = 0; i < 4; ++i) acc += rows[slot][i];
                mb_arrive(&empty[slot]);
            }
            tail += n;
            __syncwarp();
        }
        atomicAdd(out, acc);
    }
}
__global__ void probe(int variant, int rounds, int *out) {
    __shared__ int row[32];
    __shared__ uint64_t full, empty;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { mb_init(&full, 1); mb_init(&empty, 1); }
    __syncthreads();
    int acc = 0;
    if (warp == 0) {
        for (int r = 0; r < rounds; ++r) {
            if (lane == 0) {
                while (!(variant == 0 ? mb_test(&empty, (r & 1) ^ 1) : mb_try(&empty, (r & 1) ^ 1))) {}
                for (int i = 0; i < 32; ++i) row[i] = r * 32 + i;
                mb_arrive(&full);
            }
            __syncwarp();
        }
        if (variant == 2) { __syncwarp(); asm volatile("bar.sync 0;" ::: "memory"); }
        if (variant == 3) { __syncwarp(); asm volatile("bar.sync 1, 64;" ::: "memory"); }
    } else {
        for (int r = 0; r < rounds; ++r) {
            if (lane == 0) {
                while (!(variant == 0 ? mb_test(&full, r & 1) : mb_try(&full, r & 1))) {}
                for (int i = 0; i < 32; ++i) acc += row[i];
                mb_arrive(&empty);
            }
            __syncwarp();
        }
        if (variant == 2) { __syncwarp(); asm volatile("bar.sync 0;" ::: "memory"); }
        if (variant == 3) { __syncwarp(); asm volatile("bar.sync 1, 64;" ::: "memory"); }
        if (lane == 0) out[0] = acc;
    }
}
int main(int argc, char **argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    int *out; cudaMalloc(&out, 4);
    cudaMemset(out, 0, 4);
    if (variant == 4) probe_lanes<<<1, 64>>>(50, out);
    else if (variant == 5) probe_ring<<<1, 64>>>(400, out);
    else probe<<<1, 64>>>(variant, 50, out);
    cudaError_t e = cudaDeviceSynchronize();
    int h = 0; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
    printf("variant %d: %s sum %d\n", variant, cudaGetErrorString(e), h);
    return 0;
}
