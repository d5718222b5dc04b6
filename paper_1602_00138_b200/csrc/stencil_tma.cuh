// Multi-column stencil apply with TMA-staged planes (K1, the A_i W products of
// the refresh and A_i U_j of the per-RHS spaces; SchurOperator::apply,
// grid.cpp:95-97, generalised per SURVEY.md App. A).
//
// A block owns a 32 x 8 (i, j) tile of the grid for a chunk of kz planes and
// NC columns. Plane k of each column (tile + halo, 34 or 36 x 10) and of
// the four coefficient fields arrives in shared memory by ONE 4D tensor-map
// TMA load each (cp.async.bulk.tensor.4d, mbarrier completion), S stages deep,
// so HBM requests stay in flight while the block computes; out-of-grid halo
// nodes and the planes k = -1 / N2 are zero-filled by the TMA unit, which is
// exactly the Dirichlet / eliminated-Robin convention of op_prepare (every
// face coefficient toward a missing neighbour is 0). The planes k-1, k, k+1
// give y(k) with no global re-reads of x (x(k-1) at the node is carried in
// registers, so only planes k and k+1 stay resident): per node and
// column x is read from HBM once and y written once, the coefficients once per
// node for all NC columns (algorithmic bytes ncols * 2 es + 32 per node).
// Loads, products and summation order per column are those of zmarch
// (kernels.cuh), so results are bitwise identical to the one-column kernel.
#pragma once

#include "kernels.cuh"

namespace rd {

constexpr int SX = 32, SY = 8, ST_THREADS = SX * SY;
constexpr int SYH = SY + 2;  // tile rows + halo
// The box's first element along x must sit on a 16-byte boundary (a TMA load
// whose innermost start coordinate is not 16-byte aligned faults with an
// illegal instruction): float64 rows start at i0 - 2 (box 36 = 2 + 32 + 2),
// complex128 rows at i0 - 1 (box 34 x 16 B). XO = column of node i0 in the box.
template <class T> struct StX;
template <> struct StX<double> {
    static constexpr int W = 36, XO = 2;
};
template <> struct StX<cplx> {
    static constexpr int W = 34, XO = 1;
};
constexpr int SFW = 36, SFO = 2;  // coefficient fields (float64): box 36 wide from i0 - 2

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

template <class T> struct StTma {
    static constexpr uint32_t xbytes = StX<T>::W * SYH * sizeof(T);    // one column's plane tile
    static constexpr uint32_t xstride = (xbytes + 127u) & ~127u;
    static constexpr uint32_t fbytes = 4 * SFW * SYH * sizeof(double);  // the four coefficient fields
    static constexpr uint32_t fstride = (fbytes + 127u) & ~127u;
    static constexpr uint32_t stage(int nc) { return nc * xstride + fstride; }
};

// y[:, c] = A x[:, xcol ? xcol[c] : c]; blockIdx.z = (column group, k chunk).
// xmap: 4D (W*N0, N1, N2, columns of x) over doubles; fmap: 4D (N0, N1, N2, 4)
// over the (possibly row-padded) assembled fields.
// D2 (2D grids, N2 = 1): the block marches over 8-row tiles along axis 1
// instead of planes; a tile's box carries its own two halo rows, so a step
// needs only its own stage (k indexes row tiles, blockIdx.y = 0).
template <class T, int NC, bool D2>
__global__ void __launch_bounds__(ST_THREADS) stencil_tma(const __grid_constant__ CUtensorMap xmap,
                                                          const __grid_constant__ CUtensorMap fmap, OpDev op,
                                                          const int* __restrict__ xcol, T* __restrict__ y, long ldy,
                                                          int ncols, int kz, int S) {
    constexpr int W = Sc<T>::W;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[8];
    const int nk = D2 ? (op.N1 + SY - 1) / SY : op.N2;  // marched units: row tiles (2D) or planes (3D)
    const int nkc = (nk + kz - 1) / kz;
    const int cg = blockIdx.z / nkc;
    const int kc = blockIdx.z - cg * nkc;
    const int c0 = cg * NC;
    const int nc = min(NC, ncols - c0);
    const int i0 = blockIdx.x * SX, j0 = D2 ? 0 : blockIdx.y * SY;
    const int k0 = kc * kz, k1 = min(nk, k0 + kz);
    const int nplanes = D2 ? k1 - k0 : k1 - k0 + 2;  // 3D: planes k0-1 .. k1
    const uint32_t sbytes = StTma<T>::stage(NC);
    const int tid = threadIdx.x;
    int colx[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const int c = min(c0 + q, ncols - 1);
        colx[q] = xcol ? __ldg(xcol + c) : c;
    }
    auto issue = [&](int pl) {  // unit pl of the chunk into stage pl % S
        const int st = pl % S;
        unsigned char* sb = smem + (size_t)st * sbytes;
        const int kk = D2 ? 0 : k0 - 1 + pl;                // 3D: grid plane k0 - 1 + pl
        const int jb = D2 ? (k0 + pl) * SY - 1 : j0 - 1;    // 2D: rows of tile k0 + pl
        mbar_arrive_expect_tx(&full[st], nc * StTma<T>::xbytes + StTma<T>::fbytes);
        for (int q = 0; q < nc; ++q)
            tma_load_4d(sb + q * StTma<T>::xstride, &xmap, (i0 - StX<T>::XO) * W, jb, kk, colx[q], &full[st]);
        tma_load_4d(sb + NC * StTma<T>::xstride, &fmap, i0 - SFO, jb, kk, 0, &full[st]);
    };
    if (tid == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
        for (int pl = 0; pl < min(S, nplanes); ++pl) issue(pl);
    }
    __syncthreads();
    const int tx = tid % SX, ty = tid / SX;
    const int i = i0 + tx;
    int j = D2 ? k0 * SY + ty : j0 + ty;
    constexpr int XW = StX<T>::W;
    const int ci = (ty + 1) * XW + (tx + StX<T>::XO);  // x-tile index of (i, j)
    const int cf = (ty + 1) * SFW + (tx + SFO);        // field-tile index of (i, j)
    const bool three = !D2 && op.d == 3;
    const long s2 = D2 ? (long)op.N0 * SY : (long)op.N0 * op.N1;  // step of p per marched unit
    long p = i + (long)op.N0 * (j + (D2 ? 0L : (long)op.N1 * k0));
    auto wait_plane = [&](int pl) { mbar_wait(&full[pl % S], (uint32_t)(pl / S) & 1u); };
    constexpr int FP = SFW * SYH;  // field plane stride in the tile
    // 3D: x(k-1) and the -z face of plane k-1 at this node are carried in
    // registers from the previous step (as zmarch does), so plane k's stage is
    // released as soon as y(k) is done: 2 planes resident, S - 2 in flight
    T xm[NC];
    double fzm = 0.0;
    int pl = 0;  // stage of the current unit (3D: plane k; 2D: row tile k)
    if (!D2) {
        wait_plane(0);  // plane k0 - 1
        const double* F0 = reinterpret_cast<const double*>(smem + NC * StTma<T>::xstride);
        fzm = F0[3 * FP + cf];
#pragma unroll
        for (int q = 0; q < NC; ++q) xm[q] = reinterpret_cast<const T*>(smem + q * StTma<T>::xstride)[ci];
        __syncthreads();
        if (tid == 0 && S < nplanes) issue(S);
        pl = 1;
    }
    for (int k = k0; k < k1; ++k, ++pl) {
        const bool live = i < op.N0 && j < op.N1;
        wait_plane(pl);
        if (!D2) wait_plane(pl + 1);
        const unsigned char* sc = smem + (size_t)(pl % S) * sbytes;
        const unsigned char* sp = D2 ? sc : smem + (size_t)((pl + 1) % S) * sbytes;
        const double* Fc = reinterpret_cast<const double*>(sc + NC * StTma<T>::xstride);
        const double dg = Fc[cf];
        const double fxm = Fc[FP + cf - 1], fxp = Fc[FP + cf];
        const double fym = Fc[2 * FP + cf - SFW], fyp = Fc[2 * FP + cf];
        const double fzp = Fc[3 * FP + cf];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            if (q < nc) {
                const T* xk = reinterpret_cast<const T*>(sc + q * StTma<T>::xstride);
                const T xc = xk[ci];
                const T xim = xk[ci - 1], xip = xk[ci + 1], xjm = xk[ci - XW], xjp = xk[ci + XW];
                T acc = Sc<T>::zero();
                acc = axpy_real(fxm, xim, acc);
                acc = axpy_real(fxp, xip, acc);
                acc = axpy_real(fym, xjm, acc);
                acc = axpy_real(fyp, xjp, acc);
                if (three) {
                    const T xp = reinterpret_cast<const T*>(sp + q * StTma<T>::xstride)[ci];
                    acc = axpy_real(fzm, xm[q], acc);
                    acc = axpy_real(fzp, xp, acc);
                }
                const T yv = Sc<T>::sub(diag_apply<T>(dg, op.shift, xc), acc);
                if (live) y[(size_t)(c0 + q) * ldy + p] = yv;
                xm[q] = xc;
            }
        }
        fzm = fzp;
        p += s2;
        if (D2) j += SY;
        __syncthreads();  // stage pl (plane k / tile k) no longer read by anyone
        if (tid == 0 && pl + S < nplanes) issue(pl + S);
    }
}

}  // namespace rd
