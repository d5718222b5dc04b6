// Reduced-order model kernels (reference src/rom.cpp:9-67).
//
//   A_r(p) = V^T A(p) V            multi-column stencil + tiled Gram (romdot.cu)
//   A_r    = (A_r + A_r^T) / 2     rom_symmetrize
//   A_r    = P L U                 lu_pivot_col + lu_update, one column step each
//   [Y Z]  = A_r^-1 [B_r C_r]      lu_solve, one CTA per right-hand side
//   J_k    = s * vec(sum_t w_t (V Z)[i_t,:]^T (V Y)[i_t,:])   rom_jacobian
//
// The r x r factorisation is O(r^3) on a matrix that sits in L2 (r <= 1024:
// <= 16 MB complex), so a right-looking unblocked LU with one grid-wide rank-1
// update per column is enough: it is launch-bound at ~2 launches per column.
#pragma once

#include "common.cuh"

namespace rd {

// Pivot search on column k (rows k..r-1, largest modulus, ties -> smallest
// row), row interchange k <-> p over all r columns, multipliers below the
// diagonal. One CTA.
template <class T>
__global__ void __launch_bounds__(1024) lu_pivot_col(T* A, int r, int k, int* piv, int* info) {
    __shared__ double s_v[32];
    __shared__ int s_i[32];
    __shared__ int s_p;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double best = -1.0;
    int bi = r;
    for (int i = k + threadIdx.x; i < r; i += blockDim.x) {
        const double a = Sc<T>::abs2(A[(size_t)k * r + i]);
        if (a > best) {
            best = a;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
        }
    }
    if (lane == 0) {
        s_v[wid] = best;
        s_i[wid] = bi;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        best = lane < nw ? s_v[lane] : -1.0;
        bi = lane < nw ? s_i[lane] : r;
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            const bool zero = !(best > 0.0);
            s_p = zero ? k : bi;
            piv[k] = s_p;
            if (zero && *info == 0) *info = k + 1;
        }
    }
    __syncthreads();
    const int p = s_p;
    if (p != k)
        for (int j = threadIdx.x; j < r; j += blockDim.x) {
            const T t = A[(size_t)j * r + k];
            A[(size_t)j * r + k] = A[(size_t)j * r + p];
            A[(size_t)j * r + p] = t;
        }
    __syncthreads();
    const T akk = A[(size_t)k * r + k];
    if (!(Sc<T>::abs2(akk) > 0.0)) return;
    for (int i = k + 1 + threadIdx.x; i < r; i += blockDim.x) A[(size_t)k * r + i] = Sc<T>::div(A[(size_t)k * r + i], akk);
}

// Trailing rank-1 update A[k+1:, k+1:] -= A[k+1:, k] A[k, k+1:].
template <class T> __global__ void __launch_bounds__(256) lu_update(T* A, int r, int k) {
    const long m = r - k - 1;
    const long tot = m * m;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = k + 1 + (int)(e % m), j = k + 1 + (int)(e / m);
        A[(size_t)j * r + i] = Sc<T>::sub(A[(size_t)j * r + i], Sc<T>::mul(A[(size_t)k * r + i], A[(size_t)j * r + k]));
    }
}

// X[:, b] <- U^-1 L^-1 P X[:, b] for the packed LU of lu_pivot_col/lu_update;
// one CTA per column, the column staged in shared memory (r <= 2048 complex).
template <class T> __global__ void __launch_bounds__(512) lu_solve(const T* LU, int r, const int* piv, T* X, long ldx) {
    extern __shared__ unsigned char sm_raw[];
    T* x = reinterpret_cast<T*>(sm_raw);
    T* xg = X + (size_t)blockIdx.x * ldx;
    for (int i = threadIdx.x; i < r; i += blockDim.x) x[i] = xg[i];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < r; ++k) {
            const int p = piv[k];
            if (p != k) {
                const T t = x[k];
                x[k] = x[p];
                x[p] = t;
            }
        }
    __syncthreads();
    for (int k = 0; k < r; ++k) {  // unit lower
        const T xk = x[k];
        for (int i = k + 1 + threadIdx.x; i < r; i += blockDim.x)
            x[i] = Sc<T>::sub(x[i], Sc<T>::mul(LU[(size_t)k * r + i], xk));
        __syncthreads();
    }
    for (int k = r - 1; k >= 0; --k) {  // upper
        if (threadIdx.x == 0) x[k] = Sc<T>::div(x[k], LU[(size_t)k * r + k]);
        __syncthreads();
        const T xk = x[k];
        for (int i = threadIdx.x; i < k; i += blockDim.x) x[i] = Sc<T>::sub(x[i], Sc<T>::mul(LU[(size_t)k * r + i], xk));
        __syncthreads();
    }
    for (int i = threadIdx.x; i < r; i += blockDim.x) xg[i] = x[i];
}

// A <- (A + A^T) / 2 (rom.cpp:15, :25: exact symmetry of the reduced system)
template <class T> __global__ void rom_symmetrize(T* A, int r) {
    const long tot = (long)r * r;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % r), j = (int)(e / r);
        if (i >= j) continue;
        const T a = A[(size_t)j * r + i], b = A[(size_t)i * r + j];
        const T m = Sc<T>::scale(Sc<T>::add(a, b), 0.5);
        A[(size_t)j * r + i] = m;
        A[(size_t)i * r + j] = m;
    }
}

// J[d + s*nd, k] = scale * sum_{t in [ptr[k], ptr[k+1])} val[t] WZ[idx[t], d] WY[idx[t], s]
// (rom.cpp:49-63 with Wy = V Y, Wz = V Z formed once). Block y = parameter k.
template <class T>
__global__ void __launch_bounds__(256) rom_jacobian(const T* __restrict__ WY, const T* __restrict__ WZ, long n, int ns,
                                                    int nd, const long* __restrict__ ptr, const long* __restrict__ idx,
                                                    const double* __restrict__ val, double scale, T* __restrict__ J,
                                                    long ldj) {
    const int k = blockIdx.y;
    const long t0 = ptr[k], t1 = ptr[k + 1];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ns * nd; e += gridDim.x * blockDim.x) {
        const int d = e % nd, s = e / nd;
        T acc = Sc<T>::zero();
        for (long t = t0; t < t1; ++t) {
            const long i = idx[t];
            acc = Sc<T>::fma(Sc<T>::scale(WZ[(size_t)d * n + i], val[t]), WY[(size_t)s * n + i], acc);
        }
        J[(size_t)k * ldj + e] = Sc<T>::scale(acc, scale);
    }
}

}  // namespace rd
