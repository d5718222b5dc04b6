// Multi-column stencil apply with TMA-staged planes (K1, the A_i W products of
// the refresh and A_i U_j of the per-RHS spaces; SchurOperator::apply,
// grid.cpp:95-97, generalised per SURVEY.md App. A).
//
// A block owns a 32 x 8 (i, j) tile of the grid for a chunk of kz planes and
// NC columns. Plane k of each column (tile + one-node halo, 34 x 10) and of
// the four coefficient fields arrives in shared memory by ONE 4D tensor-map
// TMA load each (cp.async.bulk.tensor.4d, mbarrier completion), S stages deep,
// so HBM requests stay in flight while the block computes; out-of-grid halo
// nodes and the planes k = -1 / N2 are zero-filled by the TMA unit, which is
// exactly the Dirichlet / eliminated-Robin convention of op_prepare (every
// face coefficient toward a missing neighbour is 0). The planes k-1, k, k+1
// resident in the ring give y(k) with no global re-reads of x: per node and
// column x is read from HBM once and y written once, the coefficients once per
// node for all NC columns (algorithmic bytes ncols * 2 es + 32 per node).
// Loads, products and summation order per column are those of zmarch
// (kernels.cuh), so results are bitwise identical to the one-column kernel.
#pragma once

#include "kernels.cuh"

namespace rd {

constexpr int SX = 32, SY = 8, ST_THREADS = SX * SY;
constexpr int SXH = SX + 2, SYH = SY + 2;  // tile + halo

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

template <class T> struct StTma {
    static constexpr uint32_t xbytes = SXH * SYH * sizeof(T);          // one column's plane tile
    static constexpr uint32_t xstride = (xbytes + 127u) & ~127u;
    static constexpr uint32_t fbytes = 4 * SXH * SYH * sizeof(double);  // the four coefficient fields
    static constexpr uint32_t fstride = (fbytes + 127u) & ~127u;
    static constexpr uint32_t stage(int nc) { return nc * xstride + fstride; }
};

// y[:, c] = A x[:, xcol ? xcol[c] : c]; blockIdx.z = (column group, k chunk).
// xmap: 4D (W*N0, N1, N2, columns of x) over doubles; fmap: 4D (N0, N1, N2, 4)
// over the (possibly row-padded) assembled fields.
template <class T, int NC>
__global__ void __launch_bounds__(ST_THREADS) stencil_tma(const __grid_constant__ CUtensorMap xmap,
                                                          const __grid_constant__ CUtensorMap fmap, OpDev op,
                                                          const int* __restrict__ xcol, T* __restrict__ y, long ldy,
                                                          int ncols, int kz, int S) {
    constexpr int W = Sc<T>::W;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[8];
    const int nkc = (op.N2 + kz - 1) / kz;
    const int cg = blockIdx.z / nkc;
    const int kc = blockIdx.z - cg * nkc;
    const int c0 = cg * NC;
    const int nc = min(NC, ncols - c0);
    const int i0 = blockIdx.x * SX, j0 = blockIdx.y * SY;
    const int k0 = kc * kz, k1 = min(op.N2, k0 + kz);
    const int nplanes = k1 - k0 + 2;  // k0-1 .. k1
    const uint32_t sbytes = StTma<T>::stage(NC);
    const int tid = threadIdx.x;
    int colx[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const int c = min(c0 + q, ncols - 1);
        colx[q] = xcol ? __ldg(xcol + c) : c;
    }
    auto issue = [&](int pl) {  // plane index pl (grid plane k0 - 1 + pl) into stage pl % S
        const int st = pl % S;
        unsigned char* sb = smem + (size_t)st * sbytes;
        const int kk = k0 - 1 + pl;
        mbar_arrive_expect_tx(&full[st], nc * StTma<T>::xbytes + StTma<T>::fbytes);
        for (int q = 0; q < nc; ++q)
            tma_load_4d(sb + q * StTma<T>::xstride, &xmap, (i0 - 1) * W, j0 - 1, kk, colx[q], &full[st]);
        tma_load_4d(sb + NC * StTma<T>::xstride, &fmap, i0 - 1, j0 - 1, kk, 0, &full[st]);
    };
    if (tid == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
        for (int pl = 0; pl < min(S, nplanes); ++pl) issue(pl);
    }
    __syncthreads();
    const int tx = tid % SX, ty = tid / SX;
    const int i = i0 + tx, j = j0 + ty;
    const bool live = i < op.N0 && j < op.N1;
    const int ci = (ty + 1) * SXH + (tx + 1);  // tile-local index of (i, j)
    const bool three = op.d == 3;
    const long s2 = (long)op.N0 * op.N1;
    long p = i + (long)op.N0 * (j + (long)op.N1 * k0);
    auto wait_plane = [&](int pl) { mbar_wait(&full[pl % S], (uint32_t)(pl / S) & 1u); };
    wait_plane(0);
    wait_plane(1);
    for (int k = k0; k < k1; ++k) {
        const int pl = k - k0;  // planes pl (k-1), pl+1 (k), pl+2 (k+1)
        wait_plane(pl + 2);
        const unsigned char* sm = smem + (size_t)(pl % S) * sbytes;
        const unsigned char* sc = smem + (size_t)((pl + 1) % S) * sbytes;
        const unsigned char* sp = smem + (size_t)((pl + 2) % S) * sbytes;
        const double* Fc = reinterpret_cast<const double*>(sc + NC * StTma<T>::xstride);
        const double* Fm = reinterpret_cast<const double*>(sm + NC * StTma<T>::xstride);
        constexpr int FP = SXH * SYH;  // field plane stride in the tile
        const double dg = Fc[ci];
        const double fxm = Fc[FP + ci - 1], fxp = Fc[FP + ci];
        const double fym = Fc[2 * FP + ci - SXH], fyp = Fc[2 * FP + ci];
        const double fzm = Fm[3 * FP + ci], fzp = Fc[3 * FP + ci];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            if (q < nc) {
                const T* xk = reinterpret_cast<const T*>(sc + q * StTma<T>::xstride);
                const T xc = xk[ci];
                const T xim = xk[ci - 1], xip = xk[ci + 1], xjm = xk[ci - SXH], xjp = xk[ci + SXH];
                T acc = Sc<T>::zero();
                acc = axpy_real(fxm, xim, acc);
                acc = axpy_real(fxp, xip, acc);
                acc = axpy_real(fym, xjm, acc);
                acc = axpy_real(fyp, xjp, acc);
                if (three) {
                    const T xm = reinterpret_cast<const T*>(sm + q * StTma<T>::xstride)[ci];
                    const T xp = reinterpret_cast<const T*>(sp + q * StTma<T>::xstride)[ci];
                    acc = axpy_real(fzm, xm, acc);
                    acc = axpy_real(fzp, xp, acc);
                }
                const T yv = Sc<T>::sub(diag_apply<T>(dg, op.shift, xc), acc);
                if (live) y[(size_t)(c0 + q) * ldy + p] = yv;
            }
        }
        p += s2;
        __syncthreads();  // plane pl (k-1) no longer read by anyone
        if (tid == 0 && pl + S < nplanes) issue(pl + S);
    }
}

}  // namespace rd
