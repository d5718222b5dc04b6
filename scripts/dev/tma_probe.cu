// Stand-alone check of 4D tensor-map TMA loads (debug aid for stencil_tma.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k4(const __grid_constant__ CUtensorMap m, double* out, int c0, int c1, int c2, int c3, int bx, int by, int bz, int bw) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t bytes = bx * by * bz * bw * 8;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    const double* s = reinterpret_cast<const double*>(smem);
    for (uint32_t i = threadIdx.x; i < bytes / 8; i += blockDim.x) out[i] = s[i];
}
int main(int argc, char** argv) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    struct Case { long d0, d1, d2, d3; int b0, b1, b2, b3; int c0, c1, c2, c3; };
    Case cases[] = {{64, 30, 1, 3, 34, 10, 1, 1, -1, -1, -1, 0}, {64, 30, 1, 3, 34, 10, 1, 1, 0, 0, 0, 0},
                    {256, 128, 128, 4, 68, 10, 1, 1, -2, -1, 0, 1}, {64, 30, 1, 4, 34, 10, 1, 4, -1, -1, 0, 0},
                    {64, 30, 2, 3, 34, 10, 1, 1, 0, 0, 0, 0}, {64, 30, 2, 3, 32, 8, 1, 1, 0, 0, 0, 0},
                    {64, 30, 2, 3, 32, 8, 1, 1, 0, 0, 1, 0}, {64, 30, 2, 3, 32, 8, 1, 1, -1, 0, 0, 0},
                    {64, 30, 2, 3, 32, 8, 1, 1, 0, -1, 0, 0}, {64, 30, 2, 3, 32, 8, 1, 1, 0, 0, -1, 0},
                    {64, 30, 2, 3, 34, 8, 1, 1, 0, 0, 0, 0}, {64, 30, 2, 3, 32, 10, 1, 1, 0, 0, 0, 0},
                    {64, 30, 2, 3, 32, 8, 2, 1, 0, 0, 0, 0}, {64, 30, 2, 3, 16, 8, 1, 1, 0, 0, 0, 0}};
    const int ncase = sizeof(cases) / sizeof(cases[0]);
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    if (only < 0) { printf("%d\n", ncase); return 0; }
    for (int ci = only; ci <= only; ++ci) { auto& cs = cases[ci];
        size_t tot = cs.d0 * cs.d1 * cs.d2 * cs.d3;
        std::vector<double> h(tot);
        for (size_t i = 0; i < tot; ++i) h[i] = (double)i;
        double *d, *o;
        cudaMalloc(&d, tot * 8);
        cudaMemcpy(d, h.data(), tot * 8, cudaMemcpyHostToDevice);
        int nb = cs.b0 * cs.b1 * cs.b2 * cs.b3;
        cudaMalloc(&o, nb * 8);
        CUtensorMap m;
        cuuint64_t gd[4] = {(cuuint64_t)cs.d0, (cuuint64_t)cs.d1, (cuuint64_t)cs.d2, (cuuint64_t)cs.d3};
        cuuint64_t gs[3] = {(cuuint64_t)cs.d0 * 8, (cuuint64_t)cs.d0 * cs.d1 * 8, (cuuint64_t)cs.d0 * cs.d1 * cs.d2 * 8};
        cuuint32_t bx[4] = {(cuuint32_t)cs.b0, (cuuint32_t)cs.b1, (cuuint32_t)cs.b2, (cuuint32_t)cs.b3};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        k4<<<1, 128, nb * 8 + 256>>>(m, o, cs.c0, cs.c1, cs.c2, cs.c3, cs.b0, cs.b1, cs.b2, cs.b3);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> ho(nb);
        cudaMemcpy(ho.data(), o, nb * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int w = 0; w < cs.b3; ++w) for (int z = 0; z < cs.b2; ++z) for (int y = 0; y < cs.b1; ++y) for (int x = 0; x < cs.b0; ++x) {
            long gx = cs.c0 + x, gy = cs.c1 + y, gz = cs.c2 + z, gw = cs.c3 + w;
            double want = (gx < 0 || gy < 0 || gz < 0 || gw < 0 || gx >= cs.d0 || gy >= cs.d1 || gz >= cs.d2 || gw >= cs.d3) ? 0.0
                          : (double)(gx + cs.d0 * (gy + cs.d1 * (gz + cs.d2 * gw)));
            double got = ho[x + cs.b0 * (y + cs.b1 * (z + cs.b2 * w))];
            if (got != want) ++bad;
        }
        printf("dims %ld %ld %ld %ld box %d %d %d %d coords %d %d %d %d: encode %d kernel %s mismatches %d\n", cs.d0, cs.d1,
               cs.d2, cs.d3, cs.b0, cs.b1, cs.b2, cs.b3, cs.c0, cs.c1, cs.c2, cs.c3, (int)r, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
        cudaFree(d); cudaFree(o);
    }
    return 0;
}
