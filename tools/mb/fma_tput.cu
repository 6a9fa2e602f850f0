// Microbenchmark: FP32 FFMA vs packed FFMA2/FMUL2 issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096

__global__ void k_ffma(float *out, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < N_IT; ++i) {
        x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
        x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// 3 distinct register sources per FFMA (varying multiplicand per chain)
__global__ void k_ffma3(float *out, float a, float b) {
    float x[8], m[8], c[8];
    for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x + j; m[j] = a + j * 1e-3f; c[j] = b + j; }
    for (int i = 0; i < N_IT; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], m[j], c[j]);
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ unsigned long long pk(float a, float b) { unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__global__ void k_ffma2(float *out, float a, float b) {
    unsigned long long x[8], m = pk(a, a), c = pk(b, b);
    for (int j = 0; j < 8; ++j) x[j] = pk(threadIdx.x + j, threadIdx.x + j + 0.5f);
    for (int i = 0; i < N_IT; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[j]) : "l"(m), "l"(c));
    }
    float s = 0; for (int j = 0; j < 8; ++j) { float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(x[j])); s += p + q; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2_3(float *out, float a, float b) {
    unsigned long long x[8], m[8], c[8];
    for (int j = 0; j < 8; ++j) { x[j] = pk(threadIdx.x + j, threadIdx.x + j + 0.5f); m[j] = pk(a + j * 1e-3f, a); c[j] = pk(b + j, b); }
    for (int i = 0; i < N_IT; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[j]) : "l"(m[j]), "l"(c[j]));
    }
    float s = 0; for (int j = 0; j < 8; ++j) { float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(x[j])); s += p + q; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fmul2(float *out, float a, float b) {
    unsigned long long x[8], m = pk(a, a);
    for (int j = 0; j < 8; ++j) x[j] = pk(threadIdx.x + j, threadIdx.x + j + 0.5f);
    for (int i = 0; i < N_IT; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x[j]) : "l"(m));
    }
    float s = 0; for (int j = 0; j < 8; ++j) { float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(x[j])); s += p + q; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char *name, K k, int lanes_per_op) {
    float *d; cudaMalloc(&d, 148 * 16 * 1024 * sizeof(float));
    int blocks = 148 * 8, threads = 256;
    k<<<blocks, threads>>>(d, 0.999f, 0.001f);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(d, 0.999f, 0.001f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double inst = 5.0 * blocks * threads / 32.0 * N_IT * 8;  // warp-instructions
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-10s %8.3f ms  warp-instr/clk/SM %.3f  fp32 lane-ops/clk/SM %.1f\n", name, ms, inst / cyc / 148,
           inst * 32 * lanes_per_op / cyc / 148);
    cudaFree(d);
}
int main() {
    run("ffma", k_ffma, 1);
    run("ffma3reg", k_ffma3, 1);
    run("ffma2", k_ffma2, 2);
    run("ffma2_3reg", k_ffma2_3, 2);
    run("fmul2", k_fmul2, 2);
    return 0;
}
