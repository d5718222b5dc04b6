// Shared device helpers for the romdot B200 kernels (sm_100a).
//
// Scalars: the path computes in fp64 (real, SPD systems at omega = 0) or
// complex128 (complex-symmetric systems, omega != 0). Complex values are
// double2 {x = re, y = im}, the numpy / std::complex layout, so host buffers
// cross the C ABI unchanged.
//
// Reductions are deterministic: every block reduces its share in a fixed
// thread order, writes one partial per value, and the last block to arrive
// (atomic ticket) sums the partials in block order. No floating-point atomics.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rd {

typedef double2 cplx;

// ------------------------------------------------------------ scalar ops ---
template <class T> struct Sc;

template <> struct Sc<double> {
    static constexpr int W = 1;  // doubles per scalar
    __host__ __device__ static double zero() { return 0.0; }
    __host__ __device__ static double real(double a) { return a; }
    __host__ __device__ static double from(double a) { return a; }
    __host__ __device__ static double mul(double a, double b) { return a * b; }
    __host__ __device__ static double fma(double a, double b, double c) { return fma_(a, b, c); }
    __host__ __device__ static double cmul(double a, double b) { return a * b; }  // conj(a) * b
    __host__ __device__ static double add(double a, double b) { return a + b; }
    __host__ __device__ static double sub(double a, double b) { return a - b; }
    __host__ __device__ static double scale(double a, double s) { return a * s; }
    __host__ __device__ static double abs2(double a) { return a * a; }
    __host__ __device__ static double div(double a, double b) { return a / b; }
    __host__ __device__ static double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
        return __fma_rn(a, b, c);
#else
        return a * b + c;
#endif
    }
    __device__ static double get(const double* v) { return v[0]; }
    __device__ static void put(double* v, double a) { v[0] = a; }
};

template <> struct Sc<cplx> {
    static constexpr int W = 2;
    __host__ __device__ static cplx zero() { return make_double2(0.0, 0.0); }
    __host__ __device__ static double real(cplx a) { return a.x; }
    __host__ __device__ static cplx from(double a) { return make_double2(a, 0.0); }
    __host__ __device__ static cplx mul(cplx a, cplx b) {
        return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    }
    // c + a*b
    __host__ __device__ static cplx fma(cplx a, cplx b, cplx c) {
        return make_double2(c.x + a.x * b.x - a.y * b.y, c.y + a.x * b.y + a.y * b.x);
    }
    // conj(a) * b
    __host__ __device__ static cplx cmul(cplx a, cplx b) {
        return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
    }
    __host__ __device__ static cplx add(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
    __host__ __device__ static cplx sub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
    __host__ __device__ static cplx scale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
    __host__ __device__ static double abs2(cplx a) { return a.x * a.x + a.y * a.y; }
    __host__ __device__ static cplx div(cplx a, cplx b) {
        const double d = b.x * b.x + b.y * b.y;
        return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
    }
    __device__ static cplx get(const double* v) { return make_double2(v[0], v[1]); }
    __device__ static void put(double* v, cplx a) {
        v[0] = a.x;
        v[1] = a.y;
    }
};

// op(a) * b with op = identity (bilinear) or conj (Hermitian)
template <class T, bool HERM> __host__ __device__ inline T opmul(T a, T b) {
    return HERM ? Sc<T>::cmul(a, b) : Sc<T>::mul(a, b);
}
// acc + op(a) * b
template <class T, bool HERM> __host__ __device__ inline T opfma(T a, T b, T acc) {
    return Sc<T>::add(acc, opmul<T, HERM>(a, b));
}

__device__ inline double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-level deterministic sum of one double per thread (blockDim <= 1024).
__device__ inline double block_sum(double v, double* red /* >= 32 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    double s = 0.0;
    if (wid == 0) {
        s = lane < nw ? red[lane] : 0.0;
        s = warp_sum(s);
    }
    return s;  // valid in warp 0
}

// Grid reduction: commit this block's nv partials, return true in the last
// block. `vals` lives in shared memory and holds the block's nv values.
struct GridRed {
    double* partials;   // [gridsize][nv]
    unsigned* counter;  // zero on entry, reset by the last block
};

__device__ inline bool grid_commit(const GridRed& g, const double* vals, int nv) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) g.partials[(size_t)b * nv + v] = vals[v];
    __threadfence();
    __syncthreads();
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(g.counter, 1u);
    __syncthreads();
    return s_ticket == nb - 1;
}

// Explicit-slot variant for several independent reductions in one launch
// (the batched CG: one counter and one partial block per column): this block
// commits slot b of nb; true in the last of the nb blocks.
__device__ inline bool grid_commit_at(const GridRed& g, const double* vals, int nv, unsigned b, unsigned nb) {
    for (int v = threadIdx.x; v < nv; v += blockDim.x) g.partials[(size_t)b * nv + v] = vals[v];
    __threadfence();
    __syncthreads();
    __shared__ unsigned s_ticket2;
    if (threadIdx.x == 0) s_ticket2 = atomicAdd(g.counter, 1u);
    __syncthreads();
    return s_ticket2 == nb - 1;
}

// In the last block: out[v] = sum_b partials[b][v] in block order (fixed
// association: TPC threads per value each sum a strided block subset, then a
// fixed-order combine). Resets the counter.
__device__ inline void grid_finish(const GridRed& g, int nv, double* out /* shared or global */,
                                   unsigned nb = 0u) {
    __threadfence();
    if (nb == 0u) nb = gridDim.x * gridDim.y * gridDim.z;
    int tpc = 1;
    while (tpc * 2 * nv <= (int)blockDim.x && tpc < 32) tpc *= 2;
    const int groups = blockDim.x / tpc;
    const int sub = threadIdx.x % tpc;
    for (int v0 = 0; v0 < nv; v0 += groups) {
        const int v = v0 + threadIdx.x / tpc;
        double s = 0.0;
        if (v < nv) {
            // eight independent accumulators keep eight L2 loads in flight (a
            // single chain serialises nb / tpc round trips); fixed association
            const double* pp = g.partials + v;
            double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            unsigned b = sub;
            for (; b + 7u * tpc < nb; b += 8u * tpc) {
#pragma unroll
                for (int q = 0; q < 8; ++q) a[q] += __ldcg(pp + (size_t)(b + q * tpc) * nv);
            }
#pragma unroll
            for (int q = 0; q < 7; ++q)  // < 8 remaining slots, compile-time indices (no local memory)
                if (b + q * tpc < nb) a[q] += __ldcg(pp + (size_t)(b + q * tpc) * nv);
            s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        }
        // combine tpc lanes (tpc divides 32 and groups are lane-aligned)
        for (int o = tpc >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (v < nv && sub == 0) out[v] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *g.counter = 0u;
}

}  // namespace rd

// ------------------------------------------------ TMA bulk copy / mbarrier ---
namespace rd {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D bulk async copy global -> shared, completion counted on the mbarrier (TMA engine)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace rd
