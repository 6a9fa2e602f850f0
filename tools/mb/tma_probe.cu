// Probe: one 3-D TMA box load (cp.async.bulk.tensor) into shared memory on an mbarrier (sm_100a).
// Variants: FENCE (fence.mbarrier_init after init), GMAP (tensor map read from global memory instead of the
// kernel parameter).
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k_nob(float *out)  // mbarrier only: init, plain arrive, wait
{
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(&bar)), "r"(0) : "memory");
    if (threadIdx.x == 0) out[0] = 1.0f;
}
__global__ void k_bulk(const float *src, float *out)  // non-tensor bulk copy global -> shared
{
    __shared__ __align__(128) float buf[64];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(256) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf)), "l"(src), "r"(256), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(&bar)), "r"(0) : "memory");
    if (threadIdx.x < 64) out[threadIdx.x] = buf[threadIdx.x];
}
template <int FENCE, int GMAP>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap *gtm, float *out, int x, int y, int z, unsigned nbytes)
{
    __shared__ __align__(128) float buf[64 * 16];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
        if (FENCE) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const void *m = GMAP ? (const void *)gtm : (const void *)&tm;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(nbytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su(buf)),
                     "l"(m), "r"(x), "r"(y), "r"(z), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 360; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char **argv)
{
    const int nx = 64, ny = 64, nz = 64;
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    float *d, *o;
    CUtensorMap *g;
    cudaMalloc(&d, 4ull * nx * ny * nz);
    cudaMalloc(&o, 4 * 360);
    cudaMalloc(&g, sizeof(CUtensorMap));
    float *h = new float[nx * ny * nz];
    for (int i = 0; i < nx * ny * nz; ++i) h[i] = (float)i;
    cudaMemcpy(d, h, 4ull * nx * ny * nz, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (variant >= 6) {
        cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
        variant -= 6;
    } else {
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    }
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    CUtensorMap tm;
    cuuint64_t dims[3] = {nx, ny, nz}, str[2] = {nx * 4ull, nx * ny * 4ull};
    const int bx = getenv("BOXX") ? atoi(getenv("BOXX")) : 36, by = getenv("BOXY") ? atoi(getenv("BOXY")) : 10;
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(g, &tm, sizeof tm, cudaMemcpyHostToDevice);
    const unsigned *w32 = reinterpret_cast<const unsigned *>(&tm);
    for (int i = 0; i < 32; ++i) printf("%08x%c", w32[i], i % 8 == 7 ? '\n' : ' ');
    printf("encode %d (entry %d) variant %d\n", (int)r, (int)q, variant);
    const int X0 = getenv("X0") ? atoi(getenv("X0")) : -1;
    switch (variant) {
    case 4: k_nob<<<1, 128>>>(o); break;
    case 5: k_bulk<<<1, 128>>>(d + 64, o); break;
    case 0: k<1, 0><<<1, 128>>>(tm, g, o, X0, 3, 5, 4u * bx * by); break;
    case 1: k<0, 0><<<1, 128>>>(tm, g, o, X0, 3, 5, 4u * bx * by); break;
    case 2: k<1, 1><<<1, 128>>>(tm, g, o, X0, 3, 5, 4u * bx * by); break;
    default: k<0, 1><<<1, 128>>>(tm, g, o, X0, 3, 5, 4u * bx * by); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    float ho[360];
    cudaMemcpy(ho, o, sizeof ho, cudaMemcpyDeviceToHost);
    printf("variant %d: %s  [0]=%g [1]=%g (want 0, %g) [37]=%g (want %g)\n", variant, cudaGetErrorString(e), ho[0], ho[1],
           (float)(5 * nx * ny + 3 * nx + 0), ho[37], (float)(5 * nx * ny + 4 * nx + 0));
    return e != cudaSuccess;
}
