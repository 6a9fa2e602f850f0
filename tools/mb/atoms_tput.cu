// Microbenchmark: shared-memory integer atomics (ATOMS.ADD) throughput on sm_100a, for the
// fixed-point deposit form of the forward.  Patterns: conflict-free, "tile-like"
// (32 lanes over ~64 positions of a channel plane), same address; STS and float CAS for reference.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 2048
#define NJ 1400

__device__ __forceinline__ unsigned hsh(unsigned x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }

template <int PAT>
__global__ void k_atoms(int *out, int salt) {
    __shared__ int q[8 * NJ];
    for (int i = threadIdx.x; i < 8 * NJ; i += blockDim.x) q[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned h = hsh(threadIdx.x * 7919u + salt);
    int v = threadIdx.x;
    for (int it = 0; it < N_IT; ++it) {
        int j;
        if (PAT == 0) j = (lane + 32 * (it & 63)) ;                    // distinct banks
        else if (PAT == 1) j = (int)((h >> 3) & 63) + 64 * warp;        // 32 lanes over 64 positions
        else if (PAT == 2) j = 64 * warp;                                // one address per warp
        else j = (int)((h >> 3) & 511) + (it & 1023);                   // spread over 512
        h = h * 1664525u + 1013904223u;
#pragma unroll
        for (int c = 0; c < 7; ++c) atomicAdd(&q[c * NJ + j], v + c);
    }
    __syncthreads();
    int s = 0;
    for (int i = threadIdx.x; i < 8 * NJ; i += blockDim.x) s += q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int PAT>
__global__ void k_sts(int *out, int salt) {
    __shared__ int q[8 * NJ];
    for (int i = threadIdx.x; i < 8 * NJ; i += blockDim.x) q[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned h = hsh(threadIdx.x * 7919u + salt);
    int v = threadIdx.x;
    for (int it = 0; it < N_IT; ++it) {
        int j;
        if (PAT == 0) j = (lane + 32 * (it & 63));
        else j = (int)((h >> 3) & 63) + 64 * warp;
        h = h * 1664525u + 1013904223u;
#pragma unroll
        for (int c = 0; c < 7; ++c) { volatile int *p = &q[c * NJ + j]; *p = v + c + it; }
    }
    __syncthreads();
    int s = 0;
    for (int i = threadIdx.x; i < 8 * NJ; i += blockDim.x) s += q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fatoms(int *out, int salt) {
    __shared__ float q[8 * NJ];
    for (int i = threadIdx.x; i < 8 * NJ; i += blockDim.x) q[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    unsigned h = hsh(threadIdx.x * 7919u + salt);
    float v = threadIdx.x;
    for (int it = 0; it < N_IT / 4; ++it) {
        const int j = (int)((h >> 3) & 63) + 64 * warp;
        h = h * 1664525u + 1013904223u;
#pragma unroll
        for (int c = 0; c < 7; ++c) atomicAdd(&q[c * NJ + j], v + c);
    }
    __syncthreads();
    float s = 0;
    for (int i = threadIdx.x; i < 8 * NJ; i += blockDim.x) s += q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (int)s;
}

// 64-bit integer atomics (two 32-bit channels per word, red.shared.add.u64): 4 words per deposit
// instead of 7.  On sm_100a ptxas lowers it to a CAS loop (ATOMS.CAST.SPIN.64): there is no native
// 64-bit shared-memory add, so the deposit form stays on 32-bit words.
template <int PAT>
__global__ void k_atoms64(int *out, int salt) {
    __shared__ unsigned long long q[4 * NJ];
    for (int i = threadIdx.x; i < 4 * NJ; i += blockDim.x) q[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned h = hsh(threadIdx.x * 7919u + salt);
    unsigned long long v = threadIdx.x;
    for (int it = 0; it < N_IT; ++it) {
        int j;
        if (PAT == 0) j = (lane + 32 * (it & 63));
        else j = (int)((h >> 3) & 63) + 64 * warp;
        h = h * 1664525u + 1013904223u;
        const unsigned addr = (unsigned)__cvta_generic_to_shared(q) + 8u * (unsigned)(j * 4);  // [pos][4 words]
#pragma unroll
        for (int c = 0; c < 4; ++c)
            asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(addr + 8 * c), "l"(v + c) : "memory");
    }
    __syncthreads();
    unsigned long long s = 0;
    for (int i = threadIdx.x; i < 4 * NJ; i += blockDim.x) s += q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (int)s;
}

// the deposit form's layout: 7 u32 words per position at an odd stride, lanes at random positions
template <int PAT>
__global__ void k_atoms_dep(int *out, int salt) {
    __shared__ int q[7 * NJ];
    for (int i = threadIdx.x; i < 7 * NJ; i += blockDim.x) q[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned h = hsh(threadIdx.x * 7919u + salt);
    int v = threadIdx.x;
    for (int it = 0; it < N_IT; ++it) {
        int j;
        if (PAT == 0) j = (lane + 32 * (it & 63));
        else j = (int)((h >> 3) & 63) + 64 * warp;
        h = h * 1664525u + 1013904223u;
        const unsigned addr = (unsigned)__cvta_generic_to_shared(q) + 4u * (unsigned)(j * 7);
#pragma unroll
        for (int c = 0; c < 7; ++c) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr + 4 * c), "r"(v + c) : "memory");
    }
    __syncthreads();
    int s = 0;
    for (int i = threadIdx.x; i < 7 * NJ; i += blockDim.x) s += q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char *name, K kern, int threads, int iters_scale) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int *out;
    cudaMalloc(&out, sizeof(int) * nsm * 2 * 1024);
    const int blocks = nsm * 4;
    kern<<<blocks, threads>>>(out, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 5.0 * blocks * threads * (double)(N_IT / iters_scale) * 7;  // lane-ops
    const double per_s = ops / (ms * 1e-3);
    printf("%-28s %8.3f ms  %.3e lane-ops/s  = %.2f lane-ops/clk/SM (at %d MHz max)\n", name, ms, per_s,
           per_s / nsm / (clk * 1e3), clk / 1000);
    cudaFree(out);
}

int main() {
    run("ATOMS distinct banks", k_atoms<0>, 512, 1);
    run("ATOMS 32 lanes/64 pos", k_atoms<1>, 512, 1);
    run("ATOMS same address", k_atoms<2>, 512, 1);
    run("ATOMS spread 512", k_atoms<3>, 512, 1);
    run("dep layout u32 x7 distinct", k_atoms_dep<0>, 512, 1);
    run("dep layout u32 x7 64 pos", k_atoms_dep<1>, 512, 1);
    run("u64 x4 distinct (x7/4 scaled)", k_atoms64<0>, 512, 1);
    run("u64 x4 64 pos (x7/4 scaled)", k_atoms64<1>, 512, 1);
    run("STS distinct banks", k_sts<0>, 512, 1);
    run("STS 32 lanes/64 pos", k_sts<1>, 512, 1);
    run("float CAS 32 lanes/64 pos", k_fatoms, 512, 4);
    return 0;
}
