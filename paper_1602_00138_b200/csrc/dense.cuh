// Block kernels for the tall-skinny factorisations (sm_100a, fp64 FMA pipes):
//
//   gram_kernel     G = op(X)^T Y, X: n x a, Y: n x b  (op = T or H). 64x64
//                   (real) / 32x32 (complex) output tiles, 4x4 / 2x2 register
//                   tile per thread, row chunks staged in shared memory,
//                   deterministic split over n (slices reduced in order).
//   gemm_tall       Z = X M  or  Z = Y - X M, X: n x a, M: a x b small
//                   (device), row tiles of X staged in shared memory.
//   small dense     single-CTA Cholesky (Hermitian or bilinear), upper
//                   triangular inverse and product for the r x r factors.
//
// FP64 on B200 runs at the same rate on the FMA pipe as through DMMA, so the
// Gram products use DFMA register tiling (tcgen05 has no f64 kind).
#pragma once

#include "common.cuh"

namespace rd {

template <class T> struct GT;  // tile geometry per scalar type
// Gram block tiles (DMMA kernel below); KC is the host's slice granularity.
template <> struct GT<double> {
    static constexpr int TA = 128, TB = 128, KC = 16, WARPS_M = 4, WARPS_N = 4, THREADS = 512;
};
template <> struct GT<cplx> {
    static constexpr int TA = 64, TB = 64, KC = 16, WARPS_M = 2, WARPS_N = 4, THREADS = 256;
};

// G_partial[slice][i][j] (column-major a x b per slice) = sum_{rows in slice} op(X[r,i]) Y[r,j]
//
// FP64 tensor cores: DMMA m8n8k4 (mma.sync.aligned.m8n8k4.row.col.f64). The
// Gram is a GEMM with M = a, N = b and the long reduction K = rows: A = X^T
// (row-major in k = row, i.e. X's column-major storage), B = Y. Block tile
// TA x TB (real 128 x 128 with 16 warps as 4 x 4, complex 64 x 64 with 8
// warps as 2 x 4): per k-step of 4 rows a warp issues 16 (real) / 32
// (complex) DMMA from 8 / 12 fragment loads. Complex
// products are four real DMMA on separately staged real / imaginary planes.
// Chunks of 16 rows are staged in shared memory as [column][row] with rows
// padded to 20 (each half-warp's 16 fragment loads hit 32 distinct banks) and
// register double buffered from global memory.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

constexpr int GM_KC = 16, GM_LD = 20;

template <class T, bool HERM>
__global__ void __launch_bounds__(GT<T>::THREADS) gram_kernel(const T* __restrict__ X, long ldx, int a, const T* __restrict__ Y,
                                                   long ldy, int b, long n, long rows_per_slice, T* __restrict__ part,
                                                   bool sym_upper) {
    constexpr bool CPLX = Sc<T>::W == 2;
    constexpr int TA = GT<T>::TA, TB = GT<T>::TB, KC = GM_KC, LD = GM_LD;
    constexpr int PL = CPLX ? 2 : 1;                 // planes (re, im)
    constexpr int NTH = GT<T>::THREADS, WNN = GT<T>::WARPS_N;
    constexpr int WM = TA / GT<T>::WARPS_M, WN = TB / WNN;  // warp tile
    constexpr int MT = WM / 8, NT = WN / 8;           // mma tiles per warp
    static_assert(KC == 16, "chunk of 16 rows");
    const int ta = blockIdx.x, tb = blockIdx.y, sl = blockIdx.z;
    if (sym_upper && ta > tb) return;
    __shared__ __align__(16) double Xs[PL][TA][LD];
    __shared__ __align__(16) double Ys[PL][TB][LD];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int wm = wid / WNN, wn = wid % WNN;
    double acc[PL][MT][NT][2];
#pragma unroll
    for (int p = 0; p < PL; ++p)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[p][i][j][0] = acc[p][i][j][1] = 0.0;
    const long r0 = (long)sl * rows_per_slice;
    const long r1 = min(n, r0 + rows_per_slice);
    const int col_a0 = ta * TA, col_b0 = tb * TB;
    // global staging: 16 rows x (TA + TB) columns; thread -> (row = tid % 16, column group tid / 16)
    constexpr int CG = NTH / 16;              // column groups
    const int lr = tid & 15, lc = tid >> 4;
    constexpr int NA = TA / CG, NB = TB / CG;
    T pa[NA], pbv[NB];
    auto fetch = [&](long rc) {
        const long row = rc + lr;
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int col = col_a0 + lc + q * CG;
            pa[q] = (row < r1 && col < a) ? X[(size_t)col * ldx + row] : Sc<T>::zero();
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int col = col_b0 + lc + q * CG;
            pbv[q] = (row < r1 && col < b) ? Y[(size_t)col * ldy + row] : Sc<T>::zero();
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            if constexpr (CPLX) {
                Xs[0][lc + q * CG][lr] = ((cplx&)pa[q]).x;
                Xs[1][lc + q * CG][lr] = ((cplx&)pa[q]).y;
            } else {
                Xs[0][lc + q * CG][lr] = (double&)pa[q];
            }
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            if constexpr (CPLX) {
                Ys[0][lc + q * CG][lr] = ((cplx&)pbv[q]).x;
                Ys[1][lc + q * CG][lr] = ((cplx&)pbv[q]).y;
            } else {
                Ys[0][lc + q * CG][lr] = (double&)pbv[q];
            }
        }
    };
    const int fr = lane >> 2, fk = lane & 3;   // fragment row (m or n) and k within the step
    if (r0 < r1) fetch(r0);
    for (long rc = r0; rc < r1; rc += KC) {
        stage();
        __syncthreads();
        if (rc + KC < r1) fetch(rc + KC);
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
            double af[PL][MT], bf[PL][NT];
#pragma unroll
            for (int p = 0; p < PL; ++p) {
#pragma unroll
                for (int i = 0; i < MT; ++i) af[p][i] = Xs[p][wm * WM + i * 8 + fr][kk + fk];
#pragma unroll
                for (int j = 0; j < NT; ++j) bf[p][j] = Ys[p][wn * WN + j * 8 + fr][kk + fk];
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    if constexpr (CPLX) {
                        // T:  re += ar br - ai bi ; im += ar bi + ai br
                        // H:  re += ar br + ai bi ; im += ar bi - ai br
                        dmma(acc[0][i][j][0], acc[0][i][j][1], af[0][i], bf[0][j]);
                        dmma(acc[0][i][j][0], acc[0][i][j][1], HERM ? af[1][i] : -af[1][i], bf[1][j]);
                        dmma(acc[1][i][j][0], acc[1][i][j][1], af[0][i], bf[1][j]);
                        dmma(acc[1][i][j][0], acc[1][i][j][1], HERM ? -af[1][i] : af[1][i], bf[0][j]);
                    } else {
                        dmma(acc[0][i][j][0], acc[0][i][j][1], af[0][i], bf[0][j]);
                    }
                }
        }
        __syncthreads();
    }
    T* P = part + (size_t)sl * a * b;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int gi = col_a0 + wm * WM + i * 8 + fr;
                const int gj = col_b0 + wn * WN + j * 8 + 2 * fk + e;
                if (gi < a && gj < b) {
                    if constexpr (CPLX)
                        P[(size_t)gj * a + gi] = make_double2(acc[0][i][j][e], acc[1][i][j][e]);
                    else
                        P[(size_t)gj * a + gi] = acc[0][i][j][e];
                }
            }
}

// G = sum over slices in order; if sym, mirror the upper triangle (op(G)^T = G for
// the Hermitian case uses the conjugate).
template <class T, bool HERM>
__global__ void gram_reduce(const T* __restrict__ part, int slices, int a, int b, T* __restrict__ G, bool sym) {
    const long tot = (long)a * b;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % a), j = (int)(e / a);
        if (sym && (i / GT<T>::TA) > (j / GT<T>::TB)) {
            // lower tile: mirror from the upper element (j, i)
            T s = Sc<T>::zero();
            for (int q = 0; q < slices; ++q) s = Sc<T>::add(s, part[(size_t)q * tot + (size_t)i * a + j]);
            if constexpr (HERM) {
                if constexpr (Sc<T>::W == 2) s = make_double2(((cplx&)s).x, -((cplx&)s).y);
            }
            G[e] = s;
        } else {
            T s = Sc<T>::zero();
            for (int q = 0; q < slices; ++q) s = Sc<T>::add(s, part[(size_t)q * tot + e]);
            G[e] = s;
        }
    }
}

// Z[n x b] = (sub ? Y : 0) -/+ X[n x a] M[a x b]; M column-major (ldm = a).
// Block: 64 rows x TBc output columns; M chunk and X chunk in shared memory.
template <class T, bool SUB>
__global__ void __launch_bounds__(256) gemm_tall(const T* __restrict__ X, long ldx, int a, const T* __restrict__ M,
                                                 int b, const T* __restrict__ Y, long ldy, T* __restrict__ Z, long ldz,
                                                 long n, bool upper_tri) {
    constexpr int TR = 64;                        // rows per block
    constexpr int TC = Sc<T>::W == 1 ? 64 : 32;   // output cols per block
    constexpr int KC = 16;
    constexpr int RR = 4, RC = TC / 16;           // per-thread 4 rows x RC cols
    __shared__ T Xs[KC][TR + 1];
    __shared__ T Ms[KC][TC];
    const long row0 = (long)blockIdx.y * TR;
    const int col0 = blockIdx.x * TC;
    const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;  // 16 x 16
    T acc[RR][RC];
#pragma unroll
    for (int i = 0; i < RR; ++i)
#pragma unroll
        for (int j = 0; j < RC; ++j) acc[i][j] = Sc<T>::zero();
    const int kend = upper_tri ? min(a, col0 + TC) : a;  // M upper triangular: rows k > col are zero
    // register double buffering of the X / M chunks
    constexpr int NX = TR * KC / 256, NM = KC * TC / 256;
    T px[NX], pm[NM];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = threadIdx.x + q * 256;
            const int r = e % TR, k = e / TR;
            const long row = row0 + r;
            px[q] = (row < n && k0 + k < a) ? X[(size_t)(k0 + k) * ldx + row] : Sc<T>::zero();
        }
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            const int e = threadIdx.x + q * 256;
            const int k = e % KC, cc = e / KC;
            pm[q] = (k0 + k < a && col0 + cc < b) ? M[(size_t)(col0 + cc) * a + k0 + k] : Sc<T>::zero();
        }
    };
    if (kend > 0) fetch(0);
    for (int k0 = 0; k0 < kend; k0 += KC) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = threadIdx.x + q * 256;
            Xs[e / TR][e % TR] = px[q];
        }
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            const int e = threadIdx.x + q * 256;
            Ms[e % KC][e / KC] = pm[q];
        }
        __syncthreads();
        if (k0 + KC < kend) fetch(k0 + KC);
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            T xr[RR], mc[RC];
#pragma unroll
            for (int i = 0; i < RR; ++i) xr[i] = Xs[k][tr + 16 * i];
#pragma unroll
            for (int j = 0; j < RC; ++j) mc[j] = Ms[k][tc * RC + j];
#pragma unroll
            for (int i = 0; i < RR; ++i)
#pragma unroll
                for (int j = 0; j < RC; ++j) acc[i][j] = Sc<T>::fma(xr[i], mc[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const long row = row0 + tr + 16 * i;
        if (row >= n) continue;
#pragma unroll
        for (int j = 0; j < RC; ++j) {
            const int col = col0 + tc * RC + j;
            if (col >= b) continue;
            T v = acc[i][j];
            if (SUB) v = Sc<T>::sub(Y[(size_t)col * ldy + row], v);
            Z[(size_t)col * ldz + row] = v;
        }
    }
}

// Z[n x b] = (SUB ? Y : 0) -/+ X[n x a] M[a x b] on the FP64 tensor cores (DMMA
// m8n8k4, as gram_kernel): the MMA's M dimension is the rows of X, N the
// output columns, K the inner dimension a. Block tile 128 rows x 64 columns
// (complex: 4 real DMMA per product on split re / im planes; real: 128 x 128),
// 8 warps as 4 (rows) x 2 (columns), warp tile 32 x 32 (real 32 x 64). Chunks
// of 16 inner indices are register double buffered from global memory and
// staged as Xs[plane][k][row] (ld 136: the four k rows of an A fragment hit
// disjoint bank octets) and Ms[plane][col][k] (ld 20). upper_tri: M is upper
// triangular, so a column block stops at its last column.
constexpr int GD_TR = 128, GD_KC = 16, GD_LDX = GD_TR + 8, GD_LDM = 20;
template <class T> struct GDT;
template <> struct GDT<double> { static constexpr int TC = 128; };
template <> struct GDT<cplx> { static constexpr int TC = 64; };
template <class T> constexpr size_t gemm_dmma_smem() {
    return sizeof(double) * Sc<T>::W * (GD_KC * GD_LDX + GDT<T>::TC * GD_LDM);
}

template <class T, bool SUB>
__global__ void __launch_bounds__(256) gemm_tall_dmma(const T* __restrict__ X, long ldx, int a,
                                                      const T* __restrict__ M, int b, const T* __restrict__ Y,
                                                      long ldy, T* __restrict__ Z, long ldz, long n, bool upper_tri) {
    constexpr bool CPLX = Sc<T>::W == 2;
    constexpr int PL = CPLX ? 2 : 1;
    constexpr int TR = GD_TR, TC = GDT<T>::TC, KC = GD_KC;
    constexpr int WM = TR / 4, WN = TC / 2;  // warp tile
    constexpr int MT = WM / 8, NT = WN / 8;
    extern __shared__ __align__(16) double gd_smem[];  // Xs[PL][KC][GD_LDX], Ms[PL][TC][GD_LDM]
    auto Xs = reinterpret_cast<double (*)[KC][GD_LDX]>(gd_smem);
    auto Ms = reinterpret_cast<double (*)[TC][GD_LDM]>(gd_smem + PL * KC * GD_LDX);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int wm = wid >> 1, wn = wid & 1;
    const long row0 = (long)blockIdx.y * TR;
    const int col0 = blockIdx.x * TC;
    const int kend = upper_tri ? min(a, col0 + TC) : a;
    double acc[PL][MT][NT][2];
#pragma unroll
    for (int p = 0; p < PL; ++p)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[p][i][j][0] = acc[p][i][j][1] = 0.0;
    constexpr int NX = TR * KC / 256, NM = KC * TC / 256;
    T px[NX], pm[NM];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = tid + q * 256;
            const int r = e % TR, k = e / TR;
            const long row = row0 + r;
            px[q] = (row < n && k0 + k < kend) ? X[(size_t)(k0 + k) * ldx + row] : Sc<T>::zero();
        }
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            const int e = tid + q * 256;
            const int k = e % KC, cc = e / KC;
            pm[q] = (k0 + k < kend && col0 + cc < b) ? M[(size_t)(col0 + cc) * a + k0 + k] : Sc<T>::zero();
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = tid + q * 256;
            const int r = e % TR, k = e / TR;
            if constexpr (CPLX) {
                Xs[0][k][r] = ((cplx&)px[q]).x;
                Xs[1][k][r] = ((cplx&)px[q]).y;
            } else {
                Xs[0][k][r] = (double&)px[q];
            }
        }
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            const int e = tid + q * 256;
            const int k = e % KC, cc = e / KC;
            if constexpr (CPLX) {
                Ms[0][cc][k] = ((cplx&)pm[q]).x;
                Ms[1][cc][k] = ((cplx&)pm[q]).y;
            } else {
                Ms[0][cc][k] = (double&)pm[q];
            }
        }
    };
    const int fr = lane >> 2, fk = lane & 3;
    if (kend > 0) fetch(0);
    for (int k0 = 0; k0 < kend; k0 += KC) {
        stage();
        __syncthreads();
        if (k0 + KC < kend) fetch(k0 + KC);
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
            double af[PL][MT], bf[PL][NT];
#pragma unroll
            for (int p = 0; p < PL; ++p) {
#pragma unroll
                for (int i = 0; i < MT; ++i) af[p][i] = Xs[p][kk + fk][wm * WM + i * 8 + fr];
#pragma unroll
                for (int j = 0; j < NT; ++j) bf[p][j] = Ms[p][wn * WN + j * 8 + fr][kk + fk];
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    if constexpr (CPLX) {
                        // re += xr mr - xi mi ; im += xr mi + xi mr
                        dmma(acc[0][i][j][0], acc[0][i][j][1], af[0][i], bf[0][j]);
                        dmma(acc[0][i][j][0], acc[0][i][j][1], -af[1][i], bf[1][j]);
                        dmma(acc[1][i][j][0], acc[1][i][j][1], af[0][i], bf[1][j]);
                        dmma(acc[1][i][j][0], acc[1][i][j][1], af[1][i], bf[0][j]);
                    } else {
                        dmma(acc[0][i][j][0], acc[0][i][j][1], af[0][i], bf[0][j]);
                    }
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long row = row0 + wm * WM + i * 8 + fr;
                const int col = col0 + wn * WN + j * 8 + 2 * fk + e;
                if (row < n && col < b) {
                    T v;
                    if constexpr (CPLX)
                        v = make_double2(acc[0][i][j][e], acc[1][i][j][e]);
                    else
                        v = acc[0][i][j][e];
                    if (SUB) v = Sc<T>::sub(Y[(size_t)col * ldy + row], v);
                    Z[(size_t)col * ldz + row] = v;
                }
            }
}

// ------------------------------------------------------------ small dense ---
// In-place upper Cholesky of the r x r matrix G (column-major, ld r):
// HERM: G = S^H S ; bilinear: G = S^T S (complex symmetric). Lower part zeroed.
// info[0] = first non-positive / zero pivot index + 1 (0 = success);
// info[1] = min |S_jj|, info[2] = max |S_jj| (doubles).
template <class T> __device__ __forceinline__ T csqrt_(T v);
template <> __device__ __forceinline__ double csqrt_<double>(double v) { return sqrt(v); }
template <> __device__ __forceinline__ cplx csqrt_<cplx>(cplx v) {
    const double m = sqrt(v.x * v.x + v.y * v.y);
    double sr = sqrt(0.5 * (m + v.x));
    double si = sqrt(fmax(0.0, 0.5 * (m - v.x)));
    if (v.y < 0) si = -si;
    return make_double2(sr, si);
}
template <class T> __device__ __forceinline__ T conj_(T v);
template <> __device__ __forceinline__ double conj_<double>(double v) { return v; }
template <> __device__ __forceinline__ cplx conj_<cplx>(cplx v) { return make_double2(v.x, -v.y); }

template <class T, bool HERM>
__global__ void __launch_bounds__(1024) chol_upper(T* G, int r, double* info) {
    __shared__ T s_piv;
    __shared__ int s_bad;
    if (threadIdx.x == 0) {
        s_bad = 0;
        info[1] = 1e300;
        info[2] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < r; ++j) {
        if (threadIdx.x == 0) {
            T d = G[(size_t)j * r + j];
            bool bad;
            if (HERM || Sc<T>::W == 1) {
                const double dr = Sc<T>::real(d);
                bad = !(dr > 0.0);
                d = Sc<T>::from(bad ? 1.0 : sqrt(dr));
            } else {
                d = csqrt_<T>(d);
                bad = !(Sc<T>::abs2(d) > 0.0);
                if (bad) d = Sc<T>::from(1.0);
            }
            if (bad && !s_bad) {
                s_bad = j + 1;
                info[0] = j + 1;
            }
            const double ad = sqrt(Sc<T>::abs2(d));
            info[1] = fmin(info[1], ad);
            info[2] = fmax(info[2], ad);
            G[(size_t)j * r + j] = d;
            s_piv = d;
        }
        __syncthreads();
        const T piv = s_piv;
        // row j of S: S[j][k] = G[j][k] / piv (k > j)
        for (int k = j + 1 + threadIdx.x; k < r; k += blockDim.x)
            G[(size_t)k * r + j] = Sc<T>::div(G[(size_t)k * r + j], piv);
        __syncthreads();
        // trailing update of the upper triangle: G[k][l] -= op(S[j][k]) S[j][l], j < k <= l
        const int m = r - j - 1;
        const long tot = (long)m * (m + 1) / 2;
        for (long e = threadIdx.x; e < tot; e += blockDim.x) {
            // map e -> (k, l) with k <= l over the trailing m x m upper triangle (column-wise)
            int l = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
            while ((long)l * (l + 1) / 2 > e) --l;
            while ((long)(l + 1) * (l + 2) / 2 <= e) ++l;
            const int k = (int)(e - (long)l * (l + 1) / 2);
            const int kk = j + 1 + k, ll = j + 1 + l;
            const T sk = G[(size_t)kk * r + j], sl = G[(size_t)ll * r + j];
            G[(size_t)ll * r + kk] = Sc<T>::sub(G[(size_t)ll * r + kk], HERM ? Sc<T>::cmul(sk, sl) : Sc<T>::mul(sk, sl));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && !s_bad) info[0] = 0;
    for (long e = threadIdx.x; e < (long)r * r; e += blockDim.x) {
        const int i = (int)(e % r), jj = (int)(e / r);
        if (i > jj) G[e] = Sc<T>::zero();
    }
}

// Sinv = S^-1 for upper-triangular S (r x r, ld r); column by column.
template <class T>
__global__ void __launch_bounds__(1024) tri_inv_upper(const T* S, T* Sinv, int r) {
    for (long e = threadIdx.x; e < (long)r * r; e += blockDim.x) Sinv[e] = Sc<T>::zero();
    __syncthreads();
    for (int j = 0; j < r; ++j) {
        const T djj = Sc<T>::div(Sc<T>::from(1.0), S[(size_t)j * r + j]);
        // Sinv[i][j] = -(sum_{k=i}^{j-1} Sinv[i][k] S[k][j]) / S[j][j], i < j
        for (int i = threadIdx.x; i < j; i += blockDim.x) {
            T s = Sc<T>::zero();
            for (int k = i; k < j; ++k) s = Sc<T>::fma(Sinv[(size_t)k * r + i], S[(size_t)j * r + k], s);
            Sinv[(size_t)j * r + i] = Sc<T>::mul(Sc<T>::sub(Sc<T>::zero(), s), djj);
        }
        if (threadIdx.x == 0) Sinv[(size_t)j * r + j] = djj;
        __syncthreads();
    }
}

// C = A B for upper-triangular A, B (r x r; lda = ldb = ldc = ld), C upper.
template <class T>
__global__ void tri_mul_upper(const T* A, const T* B, T* C, int r, int ld) {
    const long tot = (long)r * r;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % r), j = (int)(e / r);
        T s = Sc<T>::zero();
        if (i <= j)
            for (int k = i; k <= j; ++k) s = Sc<T>::fma(A[(size_t)k * ld + i], B[(size_t)j * ld + k], s);
        C[(size_t)j * ld + i] = s;
    }
}

// Hermitian column norms^2 of X (n x c): out[j] = sum_i |X_ij|^2 (block partials -> last block)
template <class T>
__global__ void __launch_bounds__(256) col_norms(const T* __restrict__ X, long ldx, int c, long n, GridRed red,
                                                 double* out) {
    __shared__ double s_red[32];
    extern __shared__ double s_vals[];
    for (int j = 0; j < c; ++j) {
        double h = 0.0;
        const T* xc = X + (size_t)j * ldx;
        for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
            h += Sc<T>::abs2(xc[i]);
        const double s = block_sum(h, s_red);
        if (threadIdx.x == 0) s_vals[j] = s;
    }
    __syncthreads();
    if (!grid_commit(red, s_vals, c)) return;
    grid_finish(red, c, out);
}

}  // namespace rd

namespace rd {

// Greedy pivoted Cholesky of the Hermitian PSD Gram G (m x m, ld m), the
// column-pivoted QR pivot rule (largest residual column norm first).
// Stops when the largest remaining residual d_max <= stop_abs2 or when
// d_max <= rel_band * d0 (d0 = largest diagonal of this call).
// Outputs: piv[0..nsel), rdiag[0..nsel) = sqrt(d at pick), Rrow (mmax x m):
// Rrow[k*m + i] = R(k, i) (pivot-order row k, original column i).
// info[0] = nsel, info[1] = d_max remaining, info[2] = 1 if stopped by stop_abs2.
template <class T>
__global__ void __launch_bounds__(1024) pivoted_chol(const T* __restrict__ G, int m, double stop_abs2, double rel_band,
                                                     int* piv, double* rdiag, T* Rrow, double* info) {
    extern __shared__ double sh[];
    double* d = sh;                           // m residual norms^2
    int* picked = reinterpret_cast<int*>(d + m);  // m flags
    __shared__ double s_best[32];
    __shared__ int s_bi[32];
    __shared__ int s_p;
    __shared__ double s_dp, s_d0;
    __shared__ int s_stop;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        d[i] = Sc<T>::real(G[(size_t)i * m + i]);
        picked[i] = 0;
    }
    __syncthreads();
    int k = 0;
    for (; k < m; ++k) {
        // argmax over unpicked (deterministic: lowest index wins ties)
        double best = -1.0;
        int bi = m;
        for (int i = threadIdx.x; i < m; i += blockDim.x)
            if (!picked[i] && (d[i] > best || (d[i] == best && i < bi))) {
                best = d[i];
                bi = i;
            }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            s_best[threadIdx.x >> 5] = best;
            s_bi[threadIdx.x >> 5] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = -1.0;
            int ii = m;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
                if (s_best[w] > b || (s_best[w] == b && s_bi[w] < ii)) {
                    b = s_best[w];
                    ii = s_bi[w];
                }
            if (k == 0) s_d0 = b;
            s_stop = 0;
            if (ii >= m || b <= stop_abs2) s_stop = 2;
            else if (b <= rel_band * s_d0) s_stop = 1;
            s_p = ii;
            s_dp = b;
            info[1] = b;
            if (!s_stop) {
                piv[k] = ii;
                rdiag[k] = sqrt(b);
                picked[ii] = 1;
            }
        }
        __syncthreads();
        if (s_stop) {
            if (threadIdx.x == 0) info[2] = s_stop == 2 ? 1.0 : 0.0;
            break;
        }
        const int p = s_p;
        const double rkk = sqrt(s_dp);
        // row k: R(k, i) = (G(p, i) - sum_{l<k} conj(R(l, p)) R(l, i)) / R(k, k)
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            T v = Sc<T>::zero();
            if (i == p) {
                v = Sc<T>::from(rkk);
            } else if (!picked[i]) {
                T sum = G[(size_t)i * m + p];  // G(p, i) column-major
                for (int l = 0; l < k; ++l)
                    sum = Sc<T>::sub(sum, Sc<T>::cmul(Rrow[(size_t)l * m + p], Rrow[(size_t)l * m + i]));
                v = Sc<T>::scale(sum, 1.0 / rkk);
                d[i] -= Sc<T>::abs2(v);
            }
            Rrow[(size_t)k * m + i] = v;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) info[0] = k;
}

// dst[:, t] = src[:, idx[t]] for t < m (one launch for a whole column gather;
// blockIdx.y = t). src and dst must not overlap.
template <class T>
__global__ void gather_columns(const T* __restrict__ src, long ld, const int* __restrict__ idx, int m, long n,
                               T* __restrict__ dst, long ldd) {
    const int t = blockIdx.y;
    if (t >= m) return;
    const T* sc = src + (size_t)idx[t] * ld;
    T* dc = dst + (size_t)t * ldd;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        dc[i] = sc[i];
}

// Scale column j of X (n x c, ld) by 1/sqrt(nrm2[j]) (nrm2 = squared norms); zero columns untouched.
template <class T>
__global__ void scale_columns(T* X, long ld, int c, long n, const double* nrm2) {
    const int j = blockIdx.y;
    if (j >= c) return;
    const double s = nrm2[j] > 0.0 ? 1.0 / sqrt(nrm2[j]) : 1.0;
    T* xc = X + (size_t)j * ld;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        xc[i] = Sc<T>::scale(xc[i], s);
}

}  // namespace rd

namespace rd {

// Thin Gram G (a x b, b <= 8) = op(X)^T Y: a multi-vector T pass. Block y-index
// selects 8 CPW columns of X (CPW per warp), lanes walk rows; per-lane
// accumulators acc[CPW][b] live across the block's rows; deterministic grid
// reduction. CPW is chosen so ONE block row covers all a columns whenever the
// registers allow (a = k + 1 + appends ~ 64..81 at C4): Y is then read once,
// not once per 32-column chunk (the 32-column version re-read Y and left most
// warps of the last chunk idle: 2.9 TB/s at a = 69, b = 4).
template <class T, bool HERM, int B, int CPW>
__global__ void __launch_bounds__(256) gram_thin(const T* __restrict__ X, long ldx, int a, const T* __restrict__ Y,
                                                 long ldy, int b, long n, GridRed red, T* __restrict__ G) {
    constexpr int W = Sc<T>::W;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c0 = blockIdx.y * 8 * CPW + wid * CPW;
    T acc[CPW][B];
#pragma unroll
    for (int q = 0; q < CPW; ++q)
#pragma unroll
        for (int v = 0; v < B; ++v) acc[q][v] = Sc<T>::zero();
    for (long row = (long)blockIdx.x * 32 + lane; row < n; row += (long)gridDim.x * 32) {
        T yv[B], xv[CPW];
#pragma unroll
        for (int v = 0; v < B; ++v) yv[v] = v < b ? __ldg(Y + (size_t)v * ldy + row) : Sc<T>::zero();
#pragma unroll
        for (int q = 0; q < CPW; ++q) xv[q] = (c0 + q < a) ? __ldg(X + (size_t)(c0 + q) * ldx + row) : Sc<T>::zero();
#pragma unroll
        for (int q = 0; q < CPW; ++q)
#pragma unroll
            for (int v = 0; v < B; ++v) acc[q][v] = opfma<T, HERM>(xv[q], yv[v], acc[q][v]);
    }
    // block values: 8 CPW columns x B vectors, column-major per block chunk
    __shared__ double s_vals[8 * CPW * B * W];
#pragma unroll
    for (int q = 0; q < CPW; ++q)
#pragma unroll
        for (int v = 0; v < B; ++v) {
            double t[W];
            if constexpr (W == 1) {
                t[0] = (double&)acc[q][v];
            } else {
                t[0] = ((cplx&)acc[q][v]).x;
                t[1] = ((cplx&)acc[q][v]).y;
            }
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const double sv = warp_sum(t[w]);
                if (lane == 0) s_vals[((wid * CPW + q) * B + v) * W + w] = sv;
            }
        }
    __syncthreads();
    // grid reduction over blockIdx.x for each column chunk (blockIdx.y): reuse the
    // generic last-block sum over all blocks with a per-chunk value offset
    const int nv = 8 * CPW * B * W;
    if (!grid_commit(red, s_vals, nv)) return;
    // last block of the whole grid: sum, per chunk y, the gridDim.x partials
    __threadfence();
    const int nyc = gridDim.y;
    for (int e = threadIdx.x; e < nyc * nv; e += blockDim.x) {
        const int yc = e / nv, vv = e % nv;
        // eight independent accumulators (eight L2 loads in flight), fixed order
        const double* pp = red.partials + (size_t)gridDim.x * yc * nv + vv;
        double acc8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        unsigned bx = 0;
        for (; bx + 8 <= gridDim.x; bx += 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) acc8[q] += __ldcg(pp + (size_t)(bx + q) * nv);
        }
#pragma unroll
        for (int q = 0; q < 7; ++q)
            if (bx + q < gridDim.x) acc8[q] += __ldcg(pp + (size_t)(bx + q) * nv);
        const double sum =
            ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
        const int colr = vv / (B * W), v = (vv / W) % B, w = vv % W;
        const int col = yc * 8 * CPW + colr;
        if (col < a && v < b) reinterpret_cast<double*>(G)[((size_t)v * a + col) * W + w] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) *red.counter = 0u;
}

// Pipelined thin Gram (same result layout and reduction as gram_thin): the
// 32-row tiles of the block's 8 CPW columns of X and of the b vectors of Y are
// copied to shared memory with cp.async (16 B per thread, zero fill past the
// ends) NS stages ahead, so ~(NS-1) x 32 x (8 CPW + B) x es bytes per SM are in
// flight without costing registers (the register-staged gram_thin is
// latency-bound at ~50 KB in flight per SM). One CTA per SM; lane = row of the
// tile, warp = CPW columns, all B vectors.
template <int BYTES> __device__ __forceinline__ void cp_async_el(void* dst, const void* src, bool ok) {
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0)
                     : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <class T, bool HERM, int B, int CPW, int NS, int RT>
__global__ void __launch_bounds__(256, 1) gram_thin_pipe(const T* __restrict__ X, long ldx, int a,
                                                         const T* __restrict__ Y, long ldy, int b, long n, GridRed red,
                                                         T* __restrict__ G) {
    constexpr int W = Sc<T>::W;
    constexpr int NC = 8 * CPW;       // X columns per block
    constexpr int SE = (NC + B) * RT;  // elements per stage (RT rows per tile)
    extern __shared__ __align__(128) unsigned char gt_smem[];
    T* sm = reinterpret_cast<T*>(gt_smem);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c0b = blockIdx.y * NC;
    const long nrb = (n + RT - 1) / RT;
    const long rb0 = blockIdx.x, stride = gridDim.x;
    const long nmine = rb0 < nrb ? (nrb - rb0 + stride - 1) / stride : 0;
    auto issue = [&](long k, int stage) {
        if (k < nmine) {
            const long rb = rb0 + k * stride;
            T* st = sm + (size_t)stage * SE;
            for (int e = tid; e < SE; e += 256) {
                const int col = e / RT, rr = e % RT;
                const long row = rb * RT + rr;
                const T* src = X;
                bool ok = false;
                if (col < NC) {
                    ok = c0b + col < a && row < n;
                    if (ok) src = X + (size_t)(c0b + col) * ldx + row;
                } else {
                    ok = col - NC < b && row < n;
                    if (ok) src = Y + (size_t)(col - NC) * ldy + row;
                }
                cp_async_el<sizeof(T)>(st + e, src, ok);
            }
        }
        cp_async_commit();  // (possibly empty) group per k keeps the wait count uniform
    };
#pragma unroll
    for (int s0 = 0; s0 < NS - 1; ++s0) issue(s0, s0);
    T acc[CPW][B];
#pragma unroll
    for (int q = 0; q < CPW; ++q)
#pragma unroll
        for (int v = 0; v < B; ++v) acc[q][v] = Sc<T>::zero();
    for (long k = 0; k < nmine; ++k) {
        cp_async_wait<NS - 2>();
        __syncthreads();  // stage k landed for every thread; stage k-1 fully consumed
        issue(k + NS - 1, (int)((k + NS - 1) % NS));
        const T* st = sm + (size_t)(k % NS) * SE;
#pragma unroll
        for (int h = 0; h < RT / 32; ++h) {
            T yv[B];
#pragma unroll
            for (int v = 0; v < B; ++v) yv[v] = st[(NC + v) * RT + h * 32 + lane];
#pragma unroll
            for (int q = 0; q < CPW; ++q) {
                const T xv = st[(wid * CPW + q) * RT + h * 32 + lane];
#pragma unroll
                for (int v = 0; v < B; ++v) acc[q][v] = opfma<T, HERM>(xv, yv[v], acc[q][v]);
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    double* s_vals = reinterpret_cast<double*>(gt_smem);  // reuse the ring
#pragma unroll
    for (int q = 0; q < CPW; ++q)
#pragma unroll
        for (int v = 0; v < B; ++v) {
            double t[W];
            if constexpr (W == 1) {
                t[0] = (double&)acc[q][v];
            } else {
                t[0] = ((cplx&)acc[q][v]).x;
                t[1] = ((cplx&)acc[q][v]).y;
            }
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const double sv = warp_sum(t[w]);
                if (lane == 0) s_vals[((wid * CPW + q) * B + v) * W + w] = sv;
            }
        }
    __syncthreads();
    const int nv = NC * B * W;
    if (!grid_commit(red, s_vals, nv)) return;
    __threadfence();
    const int nyc = gridDim.y;
    for (int e = threadIdx.x; e < nyc * nv; e += blockDim.x) {
        const int yc = e / nv, vv = e % nv;
        const double* pp = red.partials + (size_t)gridDim.x * yc * nv + vv;
        double acc8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        unsigned bx = 0;
        for (; bx + 8 <= gridDim.x; bx += 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) acc8[q] += __ldcg(pp + (size_t)(bx + q) * nv);
        }
#pragma unroll
        for (int q = 0; q < 7; ++q)
            if (bx + q < gridDim.x) acc8[q] += __ldcg(pp + (size_t)(bx + q) * nv);
        const double sum =
            ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
        const int colr = vv / (B * W), v = (vv / W) % B, w = vv % W;
        const int col = yc * NC + colr;
        if (col < a && v < b) reinterpret_cast<double*>(G)[((size_t)v * a + col) * W + w] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) *red.counter = 0u;
}

// Thin GEMM Z[n x b] = Y - X M (b <= 8, X: n x a, M: a x b, ld a): thread per
// row, M in shared memory, X row read once for all b outputs.
template <class T, int B>
__global__ void __launch_bounds__(256) gemm_thin_sub(const T* __restrict__ X, long ldx, int a, const T* __restrict__ M,
                                                     int b, const T* __restrict__ Y, long ldy, T* __restrict__ Z,
                                                     long ldz, long n) {
    extern __shared__ unsigned char sm_raw[];
    T* Ms = reinterpret_cast<T*>(sm_raw);
    for (int e = threadIdx.x; e < a * b; e += blockDim.x) Ms[e] = M[e];
    __syncthreads();
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += (long)gridDim.x * blockDim.x) {
        T acc[B];
#pragma unroll
        for (int v = 0; v < B; ++v) acc[v] = Sc<T>::zero();
        for (int k = 0; k < a; ++k) {
            const T xv = X[(size_t)k * ldx + row];
#pragma unroll
            for (int v = 0; v < B; ++v)
                if (v < b) acc[v] = Sc<T>::fma(xv, Ms[(size_t)v * a + k], acc[v]);
        }
#pragma unroll
        for (int v = 0; v < B; ++v)
            if (v < b) Z[(size_t)v * ldz + row] = Sc<T>::sub(Y[(size_t)v * ldy + row], acc[v]);
    }
}

}  // namespace rd
