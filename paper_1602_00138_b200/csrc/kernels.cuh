// Device kernels of the recycled-Krylov basis build (sm_100a).
//
//  K1  stencil apply           y = A(p) x, 5/7-point variable-D Schur operator
//                              (restates SchurOperator::apply, grid.cpp:95-97,
//                              generalised per SURVEY.md App. A), multi-column
//                              with an optional column gather (A_i U_j).
//  K2  cg_stencil_dots         fused inner-iteration head: w = A r, the merged
//                              reduction {r^T r, r^T w, r^H r} and the scalar
//                              recurrence (alpha, beta, convergence, stagnation)
//                              in the last block -- one grid reduction.
//  K3  ts_T / ts_NT / ts_N     tall-skinny recycle-space projections that stream
//                              the n x c basis once per call: c = op(K)^T x,
//                              fused {x' = x - K c1 ; c2 = op(K)^T x'}, and
//                              x - K c. op = T (bilinear) or H (Hermitian).
//  K4  cg_update               q = w' - K c2 fused with the CG vector updates.
//  plus small vector kernels (norms, gathers, column scaling).
#pragma once

#include "common.cuh"

namespace rd {

// ----------------------------------------------------------- operator ---
// Coefficients are assembled once per system (op_prepare) into four node
// fields: F[0] diag (sum of face coefficients + h^2 mu_a), F[1..3] the face
// coefficient toward the +x / +y / +z neighbour (harmonic mean of the two node
// D values; 0 where the neighbour is outside the grid). The apply is then
// division-free:  y_p = (diag_p + i shift) x_p - sum_faces F_face x_q.
struct OpDev {
    int d;
    int N0, N1, N2;
    long n;
    double robin_face;  // Dbg / (1 + rho)
    double shift;       // h^2 omega/nu (imaginary diagonal)
    const double* D;    // node fields (input)
    const double* mu;
    const double* F;    // assembled [4][n]: diag, fx, fy, fz
    const double* Fp;   // the same fields with rows padded to ldF (TMA tensor maps need 16-byte row pitch)
    long ldF;           // row pitch of Fp (N0, or N0 + 1 for odd N0)
};

__device__ __forceinline__ double hmean(double a, double b) { return 2.0 * (a * b) / (a + b); }

template <class T> __device__ __forceinline__ T diag_apply(double dr, double shift, T x);
template <> __device__ __forceinline__ double diag_apply<double>(double dr, double, double x) { return dr * x; }
template <> __device__ __forceinline__ cplx diag_apply<cplx>(double dr, double s, cplx x) {
    return make_double2(dr * x.x - s * x.y, dr * x.y + s * x.x);
}
template <class T> __device__ __forceinline__ T axpy_real(double a, T x, T acc);
template <> __device__ __forceinline__ double axpy_real<double>(double a, double x, double acc) { return acc + a * x; }
template <> __device__ __forceinline__ cplx axpy_real<cplx>(double a, cplx x, cplx acc) {
    return make_double2(acc.x + a * x.x, acc.y + a * x.y);
}

// Assemble the per-system coefficient fields. Face order of the diagonal sum
// (axis 0 -, +, axis 1 -, +, axis 2 -, +) matches the CPU checker.
__global__ void __launch_bounds__(256) op_prepare(OpDev op, double* __restrict__ F) {
    const int i = blockIdx.x * 32 + (threadIdx.x & 31);
    const int j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int k = blockIdx.z;
    if (i >= op.N0 || j >= op.N1) return;
    const long s1 = op.N0, s2 = (long)op.N0 * op.N1;
    const long p = i + s1 * j + s2 * k;
    const double* D = op.D;
    const double Dp = D[p];
    const bool robin1 = (op.d == 2);
    double diag = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
    diag += (i > 0) ? hmean(Dp, D[p - 1]) : Dp;
    if (i < op.N0 - 1) {
        fx = hmean(Dp, D[p + 1]);
        diag += fx;
    } else {
        diag += Dp;
    }
    diag += (j > 0) ? hmean(Dp, D[p - s1]) : (robin1 ? op.robin_face : Dp);
    if (j < op.N1 - 1) {
        fy = hmean(Dp, D[p + s1]);
        diag += fy;
    } else {
        diag += robin1 ? op.robin_face : Dp;
    }
    if (op.d == 3) {
        diag += (k > 0) ? hmean(Dp, D[p - s2]) : op.robin_face;
        if (k < op.N2 - 1) {
            fz = hmean(Dp, D[p + s2]);
            diag += fz;
        } else {
            diag += op.robin_face;
        }
    }
    F[p] = diag + op.mu[p];
    F[op.n + p] = fx;
    F[2 * op.n + p] = fy;
    F[3 * op.n + p] = fz;
}

// Copy of the assembled fields with the row pitch rounded up to even (the
// multi-column TMA stencil's tensor map needs 16-byte row strides).
__global__ void pad_fields(const double* __restrict__ F, long n, int N0, long rows, long ldF,
                           double* __restrict__ Fp) {
    const long tot = 4 * rows * ldF;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const long f = e / (rows * ldF), rem = e - f * rows * ldF;
        const long row = rem / ldF;
        const int i = (int)(rem - row * ldF);
        Fp[e] = i < N0 ? F[f * n + row * N0 + i] : 0.0;
    }
}

// Row p of A x from the assembled fields (same face order as the checker).
template <class T>
__device__ __forceinline__ T stencil_row(const OpDev& op, const T* __restrict__ x, long p, int i, int j, int k) {
    const double* __restrict__ F = op.F;
    const long n = op.n;
    const long s1 = op.N0, s2 = (long)op.N0 * op.N1;
    T acc = Sc<T>::zero();
    if (i > 0) acc = axpy_real(__ldg(F + n + p - 1), x[p - 1], acc);
    if (i < op.N0 - 1) acc = axpy_real(__ldg(F + n + p), x[p + 1], acc);
    if (j > 0) acc = axpy_real(__ldg(F + 2 * n + p - s1), x[p - s1], acc);
    if (j < op.N1 - 1) acc = axpy_real(__ldg(F + 2 * n + p), x[p + s1], acc);
    if (op.d == 3) {
        if (k > 0) acc = axpy_real(__ldg(F + 3 * n + p - s2), x[p - s2], acc);
        if (k < op.N2 - 1) acc = axpy_real(__ldg(F + 3 * n + p), x[p + s2], acc);
    }
    return Sc<T>::sub(diag_apply<T>(__ldg(F + p), op.shift, x[p]), acc);
}

// 3D launch: block 32 x 8 threads covers an (i, j) tile, blockIdx.z = k.
__device__ __forceinline__ bool node_of_block(const OpDev& op, int& i, int& j, int& k, long& p) {
    i = blockIdx.x * 32 + (threadIdx.x & 31);
    j = blockIdx.y * 8 + (threadIdx.x >> 5);
    k = blockIdx.z;
    p = i + (long)op.N0 * (j + (long)op.N1 * k);
    return i < op.N0 && j < op.N1;
}

__device__ __forceinline__ void node_coords(const OpDev& op, long p, int& i, int& j, int& k) {
    const int pi = (int)p;
    i = pi % op.N0;
    const int q = pi / op.N0;
    j = q % op.N1;
    k = q / op.N1;
}

// y[:, c] = A x[:, xcol ? xcol[c] : c] for c < ncols. One thread per node
// (32 x 8 (i, j) tile per block, blockIdx.z = k); the node's seven
// coefficients are loaded once and applied to every column.
template <class T>
__global__ void __launch_bounds__(256) stencil_kernel(OpDev op, const T* __restrict__ x, long ldx,
                                                      const int* __restrict__ xcol, T* __restrict__ y, long ldy,
                                                      int ncols, int kz);

// z-marching stencil sweep for one (i, j) column over planes [k0, k1): x at
// k-1, k, k+1 and the -z face coefficient stay in registers from plane to
// plane, so each plane loads x(k+1), four in-plane x neighbours and six
// coefficients (the +x/+y/+z/diag of p and the -x/-y faces of the neighbours).
// f(p, xc, y) is called per plane with the row result y = (A x)_p.
template <class T, class F>
__device__ __forceinline__ void zmarch(const OpDev& op, const T* __restrict__ x, int i, int j, int k0, int k1, F&& f) {
    const long n = op.n;
    const long s1 = op.N0, s2 = (long)op.N0 * op.N1;
    const double* __restrict__ Fd = op.F;
    long p = i + s1 * (j + (long)op.N1 * k0);
    const bool three = op.d == 3;
    T xm = (three && k0 > 0) ? x[p - s2] : Sc<T>::zero();
    double fzm = (three && k0 > 0) ? __ldg(Fd + 3 * n + p - s2) : 0.0;
    T xc = x[p];
    const bool hx_m = i > 0, hx_p = i < op.N0 - 1, hy_m = j > 0, hy_p = j < op.N1 - 1;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
        const bool hz_p = three && k < op.N2 - 1;
        const T xp = hz_p ? x[p + s2] : Sc<T>::zero();
        const double fzp = hz_p ? __ldg(Fd + 3 * n + p) : 0.0;
        const double dg = __ldg(Fd + p);
        const double fxm = hx_m ? __ldg(Fd + n + p - 1) : 0.0;
        const double fxp = hx_p ? __ldg(Fd + n + p) : 0.0;
        const double fym = hy_m ? __ldg(Fd + 2 * n + p - s1) : 0.0;
        const double fyp = hy_p ? __ldg(Fd + 2 * n + p) : 0.0;
        const T xim = hx_m ? x[p - 1] : Sc<T>::zero();
        const T xip = hx_p ? x[p + 1] : Sc<T>::zero();
        const T xjm = hy_m ? x[p - s1] : Sc<T>::zero();
        const T xjp = hy_p ? x[p + s1] : Sc<T>::zero();
        T acc = Sc<T>::zero();
        acc = axpy_real(fxm, xim, acc);
        acc = axpy_real(fxp, xip, acc);
        acc = axpy_real(fym, xjm, acc);
        acc = axpy_real(fyp, xjp, acc);
        if (three) {
            acc = axpy_real(fzm, xm, acc);
            acc = axpy_real(fzp, xp, acc);
        }
        const T yv = Sc<T>::sub(diag_apply<T>(dg, op.shift, xc), acc);
        f(p, xc, yv);
        xm = xc;
        xc = xp;
        fzm = fzp;
        p += s2;
    }
}

// y[:, c] = A x[:, xcol ? xcol[c] : c]: blockIdx.z = (column, k chunk of kz planes)
template <class T>
__global__ void __launch_bounds__(256) stencil_kernel(OpDev op, const T* __restrict__ x, long ldx,
                                                      const int* __restrict__ xcol, T* __restrict__ y, long ldy,
                                                      int ncols, int kz) {
    const int nkc = (op.N2 + kz - 1) / kz;
    const int c = blockIdx.z / nkc;
    const int kc = blockIdx.z - c * nkc;
    const int i = blockIdx.x * 32 + (threadIdx.x & 31);
    const int j = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (c >= ncols || i >= op.N0 || j >= op.N1) return;
    const int k0 = kc * kz, k1 = min(op.N2, k0 + kz);
    const T* xc = x + (size_t)(xcol ? xcol[c] : c) * ldx;
    T* yc = y + (size_t)c * ldy;
    zmarch<T>(op, xc, i, j, k0, k1, [&](long p, const T&, const T& v) { yc[p] = v; });
}

// Multi-column apply, NC columns per thread: the node's coefficients are loaded
// once per plane and applied to all NC columns (the one-column kernel above
// re-reads them per column: 0.36-0.55 of HBM peak at 8 columns in the C5 sweep).
// Same loads and summation order per column as zmarch.
template <class T, int NC>
__global__ void __launch_bounds__(256) stencil_kernel_mc(OpDev op, const T* __restrict__ x, long ldx,
                                                         const int* __restrict__ xcol, T* __restrict__ y, long ldy,
                                                         int ncols, int kz) {
    const int nkc = (op.N2 + kz - 1) / kz;
    const int cg = blockIdx.z / nkc;
    const int kc = blockIdx.z - cg * nkc;
    const int i = blockIdx.x * 32 + (threadIdx.x & 31);
    const int j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int c0 = cg * NC;
    if (c0 >= ncols || i >= op.N0 || j >= op.N1) return;
    const int k0 = kc * kz, k1 = min(op.N2, k0 + kz);
    const long n = op.n;
    const long s1 = op.N0, s2 = (long)op.N0 * op.N1;
    const double* __restrict__ Fd = op.F;
    const bool three = op.d == 3;
    const T* xs[NC];
    T* ys[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const int c = min(c0 + q, ncols - 1);
        xs[q] = x + (size_t)(xcol ? xcol[c] : c) * ldx;
        ys[q] = y + (size_t)(c0 + q) * ldy;
    }
    long p = i + s1 * (j + (long)op.N1 * k0);
    T xm[NC], xc[NC];
    double fzm = (three && k0 > 0) ? __ldg(Fd + 3 * n + p - s2) : 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        xm[q] = (three && k0 > 0) ? xs[q][p - s2] : Sc<T>::zero();
        xc[q] = xs[q][p];
    }
    const bool hx_m = i > 0, hx_p = i < op.N0 - 1, hy_m = j > 0, hy_p = j < op.N1 - 1;
    for (int k = k0; k < k1; ++k) {
        const bool hz_p = three && k < op.N2 - 1;
        const double fzp = hz_p ? __ldg(Fd + 3 * n + p) : 0.0;
        const double dg = __ldg(Fd + p);
        const double fxm = hx_m ? __ldg(Fd + n + p - 1) : 0.0;
        const double fxp = hx_p ? __ldg(Fd + n + p) : 0.0;
        const double fym = hy_m ? __ldg(Fd + 2 * n + p - s1) : 0.0;
        const double fyp = hy_p ? __ldg(Fd + 2 * n + p) : 0.0;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const T* xq = xs[q];
            const T xp = hz_p ? xq[p + s2] : Sc<T>::zero();
            const T xim = hx_m ? xq[p - 1] : Sc<T>::zero();
            const T xip = hx_p ? xq[p + 1] : Sc<T>::zero();
            const T xjm = hy_m ? xq[p - s1] : Sc<T>::zero();
            const T xjp = hy_p ? xq[p + s1] : Sc<T>::zero();
            T acc = Sc<T>::zero();
            acc = axpy_real(fxm, xim, acc);
            acc = axpy_real(fxp, xip, acc);
            acc = axpy_real(fym, xjm, acc);
            acc = axpy_real(fyp, xjp, acc);
            if (three) {
                acc = axpy_real(fzm, xm[q], acc);
                acc = axpy_real(fzp, xp, acc);
            }
            const T yv = Sc<T>::sub(diag_apply<T>(dg, op.shift, xc[q]), acc);
            if (c0 + q < ncols) ys[q][p] = yv;
            xm[q] = xc[q];
            xc[q] = xp;
        }
        fzm = fzp;
        p += s2;
    }
}

// ------------------------------------------------------------ CG state ---
// Scalars of one recycled CG / COCG solve (Chronopoulos-Gear recurrence).
struct CGState {
    double2 alpha, beta, alpha_prev, gamma_prev, gamma;
    double scale, tol, best, relres;
    int it, maxit, stagnant, done, converged, hist_cap, pad0, pad1;
};

template <class T> __device__ __forceinline__ T ld2(double2 v);
template <> __device__ __forceinline__ double ld2<double>(double2 v) { return v.x; }
template <> __device__ __forceinline__ cplx ld2<cplx>(double2 v) { return v; }
template <class T> __device__ __forceinline__ double2 st2(T v);
template <> __device__ __forceinline__ double2 st2<double>(double v) { return make_double2(v, 0.0); }
template <> __device__ __forceinline__ double2 st2<cplx>(cplx v) { return v; }

__device__ inline bool finite_(double v) { return isfinite(v); }

// Chronopoulos-Gear scalar step of one CG / COCG solve from the merged
// reduction s_tot = {r^T r (W), r^T A r (W), r^H r}: convergence, the 1000-step
// stagnation window, then alpha / beta. Runs in one thread.
template <class T>
__device__ __noinline__ void cg_recurrence(CGState* st, const double* s_tot, double* hist) {
    constexpr int W = Sc<T>::W;
    T gamma, delta;
    if constexpr (W == 1) {
        gamma = s_tot[0];
        delta = s_tot[1];
    } else {
        gamma = make_double2(s_tot[0], s_tot[1]);
        delta = make_double2(s_tot[2], s_tot[3]);
    }
    const double rho2 = s_tot[2 * W];
    const int it = st->it;
    const double relres = st->scale > 0.0 ? sqrt(rho2) / st->scale : 0.0;
    st->relres = relres;
    if (hist && it < st->hist_cap) hist[it] = relres;
    if (it == 0) {
        st->best = relres;
        if (rho2 == 0.0 || st->scale == 0.0 || relres <= st->tol) {
            st->converged = 1;
            st->done = 1;
            return;
        }
    } else {
        if (!finite_(relres)) {
            st->done = 1;
            return;
        }
        if (relres <= st->tol) {
            st->converged = 1;
            st->done = 1;
            return;
        }
        // CG residuals are not monotone: 1000-step window (the reference's 50 is for MINRES)
        if (relres < st->best * (1.0 - 1e-12)) {
            st->best = relres;
            st->stagnant = 0;
        } else if (++st->stagnant >= 1000) {
            st->done = 1;
            return;
        }
    }
    if (it >= st->maxit) {
        st->done = 1;
        return;
    }
    T alpha, beta;
    if (it == 0) {
        beta = Sc<T>::zero();
        alpha = Sc<T>::div(gamma, delta);
    } else {
        const T gp = ld2<T>(st->gamma_prev), ap = ld2<T>(st->alpha_prev);
        beta = Sc<T>::div(gamma, gp);
        alpha = Sc<T>::div(gamma, Sc<T>::sub(delta, Sc<T>::div(Sc<T>::mul(beta, gamma), ap)));
    }
    st->alpha = st2<T>(alpha);
    st->beta = st2<T>(beta);
    st->gamma = st2<T>(gamma);
}

// K2: w = A r ; partials of {r^T r (W), r^T w (W), r^H r (1)} ; last block runs
// the scalar recurrence. One grid reduction per iteration.
template <class T>
__global__ void __launch_bounds__(256) cg_stencil_dots(OpDev op, const T* __restrict__ r, T* __restrict__ w,
                                                       CGState* st, double* hist, GridRed red, int kz) {
    if (st->done) return;
    constexpr int W = Sc<T>::W;
    T g = Sc<T>::zero(), dl = Sc<T>::zero();
    double h = 0.0;
    // block = (32 x 8) x-y tile marching over kz planes (blockIdx.z chunk)
    const int i = blockIdx.x * 32 + (threadIdx.x & 31);
    const int j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int k0 = blockIdx.z * kz, k1 = min(op.N2, k0 + kz);
    if (i < op.N0 && j < op.N1)
        zmarch<T>(op, r, i, j, k0, k1, [&](long p, const T& rp, const T& wp) {
            w[p] = wp;
            g = Sc<T>::fma(rp, rp, g);
            dl = Sc<T>::fma(rp, wp, dl);
            h += Sc<T>::abs2(rp);
        });
    __shared__ double s_red[32];
    __shared__ double s_vals[2 * W + 1];
    double v[2 * W + 1];
    if constexpr (W == 1) {
        v[0] = g;
        v[1] = dl;
        v[2] = h;
    } else {
        v[0] = ((cplx&)g).x;
        v[1] = ((cplx&)g).y;
        v[2] = ((cplx&)dl).x;
        v[3] = ((cplx&)dl).y;
        v[4] = h;
    }
#pragma unroll
    for (int t = 0; t < 2 * W + 1; ++t) {
        const double s = block_sum(v[t], s_red);
        if (threadIdx.x == 0) s_vals[t] = s;
    }
    __syncthreads();
    if (!grid_commit(red, s_vals, 2 * W + 1)) return;
    __shared__ double s_tot[2 * W + 1];
    grid_finish(red, 2 * W + 1, s_tot);
    if (threadIdx.x != 0) return;
    cg_recurrence<T>(st, s_tot, hist);
}

// Batched CG update, blockIdx.y = column: p = r + beta p ; s = w + beta s ;
// y += alpha p ; r -= alpha s (thread per row).
template <class T>
__global__ void __launch_bounds__(256) bcg_update(T* __restrict__ R, T* __restrict__ Pv, T* __restrict__ S,
                                                  T* __restrict__ Y, const T* __restrict__ Wv, long ld, long n,
                                                  CGState* st) {
    const int c = blockIdx.y;
    CGState* sc = st + c;
    if (sc->done) return;
    const T alpha = ld2<T>(sc->alpha), beta = ld2<T>(sc->beta);
    const size_t off = (size_t)c * ld;
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += (long)gridDim.x * blockDim.x) {
        const T rv = R[off + row];
        const T pn = Sc<T>::fma(beta, Pv[off + row], rv);
        const T sn = Sc<T>::fma(beta, S[off + row], Wv[off + row]);
        Pv[off + row] = pn;
        S[off + row] = sn;
        Y[off + row] = Sc<T>::fma(alpha, pn, Y[off + row]);
        R[off + row] = Sc<T>::sub(rv, Sc<T>::mul(alpha, sn));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->gamma_prev = sc->gamma;
        sc->alpha_prev = sc->alpha;
        sc->it = sc->it + 1;
    }
}

// Selective reorthogonalisation (Kahan-Parlett "twice is enough"): when the
// first CGS pass keeps at least half of ||z||^2 (||q1||^2 >= ||z||^2 / 2,
// both measured) it is already accurate to O(eps) and the second pass is
// skipped: flag->done = 1 (the second-pass kernels then exit at entry) and
// c2 = 0. Otherwise flag->done = 0 and the second pass runs. The measured
// ||q1|| keeps the test valid for bilinear (complex K^T K = I) spaces too.
__global__ void reorth_decide(const double* __restrict__ nrmq, const double* __restrict__ nrmz, int nv, double* c2,
                              CGState* flag) {
    __shared__ int s_skip;
    if (threadIdx.x == 0) {
        s_skip = (nrmq[0] >= 0.5 * nrmz[0]) ? 1 : 0;
        flag->done = s_skip;
    }
    __syncthreads();
    if (s_skip)
        for (int i = threadIdx.x; i < nv; i += blockDim.x) c2[i] = 0.0;
}

// Symmetric Gram of a per-RHS recycle space K = [Q0 Kt] (c = ku + m columns):
// G[:ku, :ku] = G00 (the system's eigen block, ld ku), G[:, ku:] = Gt (c x m,
// ld c), G[ku:, :ku] = Gt[:ku, :]^T (bilinear: no conjugation).
template <class T>
__global__ void assemble_space_gram(const T* __restrict__ G00, int ku, const T* __restrict__ Gt, int c,
                                    T* __restrict__ G) {
    const long tot = (long)c * c;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % c), j = (int)(e / c);
        T v;
        if (j >= ku)
            v = Gt[(size_t)(j - ku) * c + i];
        else if (i >= ku)
            v = Gt[(size_t)(i - ku) * c + j];
        else
            v = G00[(size_t)j * ku + i];
        G[e] = v;
    }
}

// X <- X S for a small upper-triangular S (m x m, column-major, ld m) staged in
// shared memory: thread per row, the row's MW leading entries in registers, in
// place. The CholQR step of the per-RHS trailing block (X = Kt or Ut, S = the
// inverse of the bilinear Cholesky factor of Kt^T Kt).
template <class T, int MW>
__global__ void __launch_bounds__(256) tri_right_inplace(T* __restrict__ X, long ld, int m, const T* __restrict__ S,
                                                         long n) {
    __shared__ T s_S[MW * MW];
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) s_S[e] = S[e];
    __syncthreads();
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += (long)gridDim.x * blockDim.x) {
        T x[MW];
#pragma unroll
        for (int i = 0; i < MW; ++i) x[i] = i < m ? X[(size_t)i * ld + row] : Sc<T>::zero();
#pragma unroll
        for (int j = MW - 1; j >= 0; --j) {
            if (j < m) {
                T y = Sc<T>::zero();
#pragma unroll
                for (int i = 0; i <= j; ++i) y = Sc<T>::fma(x[i], s_S[j * m + i], y);
                X[(size_t)j * ld + row] = y;
            }
        }
    }
}

// Gt (cj x m, ld cj) = [Ce ; Gtt]: Ce = Kb^T Kt (ku x m, ld ku), Gtt = Kt^T Kt (m x m).
template <class T>
__global__ void stack_space_gt(const T* __restrict__ Ce, int ku, const T* __restrict__ Gtt, int m,
                               T* __restrict__ Gt) {
    const int cj = ku + m;
    const long tot = (long)cj * m;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % cj), q = (int)(e / cj);
        Gt[e] = i < ku ? Ce[(size_t)q * ku + i] : Gtt[(size_t)q * m + (i - ku)];
    }
}

// One-pass CGS coefficient against the eigen block (Gram-corrected, as the
// inner iteration's): Co = 2 C1 - G00 C1, G00 = Kb^T Kb (ku x ku), C1 = Kb^T Kt
// (ku x m, ld ku); Kt - Kb Co equals the two-pass CGS in exact arithmetic.
template <class T>
__global__ void onepass_coef(const T* __restrict__ G00, int ku, const T* __restrict__ C1, int m, T* __restrict__ Co) {
    const long tot = (long)ku * m;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % ku), t = (int)(e / ku);
        T acc = Sc<T>::zero();
        for (int k = 0; k < ku; ++k) acc = Sc<T>::fma(G00[(size_t)k * ku + i], C1[(size_t)t * ku + k], acc);
        Co[e] = Sc<T>::sub(Sc<T>::scale(C1[e], 2.0), acc);
    }
}

// R[idx[c] + c*ld] = val[c] (unit right-hand sides of the layout)
template <class T>
__global__ void scatter_unit_rhs(T* R, long ld, const long* __restrict__ idx, const double* __restrict__ val, int m) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < m) R[(size_t)c * ld + idx[c]] = Sc<T>::from(val[c]);
}

// ------------------------------------------------- tall-skinny passes ---
// Tile = 32 rows (one per lane); warp w of the 8 owns columns
// [w*CPW, (w+1)*CPW) of the current column chunk. Per-lane accumulators live
// across the block's grid-stride tiles; one warp reduction at the end.
constexpr int TS_THREADS = 256;
constexpr int TS_WARPS = 8;

// Batched streaming loads: volatile PTX loads keep their program order, and the
// empty volatile "fence" that names every loaded register makes the consumer
// FMAs wait until all loads of the batch have been issued (ILP, not one load
// in flight per thread).
template <class T> __device__ __forceinline__ T ldg_nc(const T* p);
// Coherent (L2) loads: these kernels may write another column of the same
// allocation in place, so the non-coherent texture path is not used.
template <> __device__ __forceinline__ double ldg_nc<double>(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
template <> __device__ __forceinline__ cplx ldg_nc<cplx>(const cplx* p) {
    cplx v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <class T> __device__ __forceinline__ void reg_fence(T& v);
template <> __device__ __forceinline__ void reg_fence<double>(double& v) { asm volatile("" : "+d"(v)); }
template <> __device__ __forceinline__ void reg_fence<cplx>(cplx& v) { asm volatile("" : "+d"(v.x), "+d"(v.y)); }

// Basis addressing. Column-major: (i, j) -> j*ld + i. Row-blocked ("RB"):
// 32-row blocks, each holding all C columns contiguously,
// (i, j) -> (i/32)*32*C + j*32 + i%32, so every 32-row tile of the basis the
// inner-iteration kernels touch is one contiguous chunk of 32*C elements.
template <bool RB> __device__ __forceinline__ size_t kaddr(long row, int j, long ld) {
    if (RB) return (size_t)(row >> 5) * (32 * (size_t)ld) + (size_t)j * 32 + (size_t)(row & 31);
    return (size_t)j * ld + (size_t)row;
}

// Repack an n x c column-major basis into the row-blocked layout (zero pad).
template <class T>
__global__ void repack_rb(const T* __restrict__ K, long ldk, int c, long n, T* __restrict__ out, long nrows_out) {
    const long nb = (nrows_out + 31) >> 5;
    const long tot = nb * 32 * (long)c;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const long rb = e / (32L * c);
        const long rem = e - rb * 32L * c;
        const int j = (int)(rem >> 5);
        const long row = rb * 32 + (rem & 31);
        out[e] = row < n ? K[(size_t)j * ldk + row] : Sc<T>::zero();
    }
}

template <class T, bool HERM, int CPW>
__device__ __forceinline__ void ts_finish_cols(T (&acc)[CPW], int c, int col0, GridRed red, double* out,
                                               const double* flagdone) {
    constexpr int W = Sc<T>::W;
    __shared__ double s_vals[TS_WARPS * CPW * W];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
        double a[W];
        if constexpr (W == 1) {
            a[0] = (double&)acc[jj];
        } else {
            a[0] = ((cplx&)acc[jj]).x;
            a[1] = ((cplx&)acc[jj]).y;
        }
#pragma unroll
        for (int t = 0; t < W; ++t) {
            const double s = warp_sum(a[t]);
            if (lane == 0) s_vals[(wid * CPW + jj) * W + t] = s;
        }
    }
    __syncthreads();
    const int nv = c * W;
    if (!grid_commit(red, s_vals, nv)) return;
    grid_finish(red, nv, out + (size_t)col0 * W);
}

// Rows per lane per step: enough independent loads in flight per lane
// (CPW columns x U rows) to cover HBM latency.
template <class T, int CPW> struct TSU {
    static constexpr int LOADS = Sc<T>::W == 1 ? 16 : 8;
    static constexpr int U = CPW >= LOADS ? 1 : (LOADS / CPW > 8 ? 8 : LOADS / CPW);
};

// out[col0 + j] = sum_i op(K[i, col0 + j]) x[i], j < c (c <= 8*CPW)
// Loads use clamped (always valid) indices so every lane issues all CPW x U
// loads back to back; out-of-range rows are masked through x = 0 and
// out-of-range columns are never committed.
template <class T, bool HERM, int CPW, bool RB>
__global__ void __launch_bounds__(TS_THREADS) ts_T(const T* __restrict__ K, long ldk, int c, int col0,
                                                   const T* __restrict__ x, long n, GridRed red, double* out,
                                                   const CGState* st) {
    if (st && st->done) return;
    constexpr int U = TSU<T, CPW>::U;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int j0 = wid * CPW;
    T acc[CPW];
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) acc[jj] = Sc<T>::zero();
    int ncol = c - j0;
    if (ncol > CPW) ncol = CPW;
    if (ncol < 1) ncol = 1;
    const int jbase = (j0 < c ? j0 : 0) + col0;
    const long nsteps = (n + 32 * U - 1) / (32 * U);
    for (long stp = blockIdx.x; stp < nsteps; stp += gridDim.x) {
        const long base = stp * 32 * U + lane;
        T xv[U];
        T kv[U][CPW];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long row = base + 32 * u;
            const long rr = row < n ? row : n - 1;
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) kv[u][jj] = ldg_nc(K + kaddr<RB>(rr, jbase + (jj < ncol ? jj : ncol - 1), ldk));
            xv[u] = ldg_nc(x + rr);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) reg_fence(kv[u][jj]);
            reg_fence(xv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + 32 * u >= n) xv[u] = Sc<T>::zero();
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) acc[jj] = opfma<T, HERM>(kv[u][jj], xv[u], acc[jj]);
        }
    }
    ts_finish_cols<T, HERM, CPW>(acc, c, col0, red, out, nullptr);
}

// Fused CGS pass: xo = x - K c1 (c1 = cin, device), out = op(K)^T xo.
template <class T, bool HERM, int CPW, bool RB>
__global__ void __launch_bounds__(TS_THREADS) ts_NT(const T* __restrict__ K, long ldk, int c,
                                                    const T* x, T* xo, long n,
                                                    const double* __restrict__ cin, GridRed red, double* out,
                                                    const CGState* st) {
    if (st && st->done) return;
    constexpr int W = Sc<T>::W;
    constexpr int U = TSU<T, CPW>::U;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int j0 = wid * CPW;
    __shared__ T s_part[TS_WARPS][32 * U];
    __shared__ T s_cw[TS_WARPS * CPW];
    for (int t = threadIdx.x; t < TS_WARPS * CPW; t += blockDim.x)
        s_cw[t] = t < c ? Sc<T>::get(cin + (size_t)t * W) : Sc<T>::zero();
    __syncthreads();
    int ncol = c - j0;
    if (ncol > CPW) ncol = CPW;
    if (ncol < 1) ncol = 1;
    const int jbase = j0 < c ? j0 : 0;
    T acc[CPW];
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) acc[jj] = Sc<T>::zero();
    const long nsteps = (n + 32 * U - 1) / (32 * U);
    for (long stp = blockIdx.x; stp < nsteps; stp += gridDim.x) {
        const long base = stp * 32 * U + lane;
        T xv[U];
        T kv[U][CPW];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long row = base + 32 * u;
            const long rr = row < n ? row : n - 1;
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) kv[u][jj] = ldg_nc(K + kaddr<RB>(rr, jbase + (jj < ncol ? jj : ncol - 1), ldk));
            // xo may alias x (in-place CGS2) and every warp consumes x[row] after the
            // barrier while warp 0 stores xo[row]: the load must stay before the
            // barrier (volatile coherent load + register fence; no __restrict__ on
            // x/xo, which would license a non-coherent reload after it).
            xv[u] = ldg_nc(x + rr);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            reg_fence(xv[u]);
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) reg_fence(kv[u][jj]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            T part = Sc<T>::zero();
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) part = Sc<T>::fma(kv[u][jj], s_cw[j0 + jj], part);
            s_part[wid][32 * u + lane] = part;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < U; ++u) {
            T sum = s_part[0][32 * u + lane];
#pragma unroll
            for (int w2 = 1; w2 < TS_WARPS; ++w2) sum = Sc<T>::add(sum, s_part[w2][32 * u + lane]);
            const long row = base + 32 * u;
            T xn = Sc<T>::sub(xv[u], sum);
            if (row >= n) xn = Sc<T>::zero();
            if (wid == 0 && row < n) xo[row] = xn;
#pragma unroll
            for (int jj = 0; jj < CPW; ++jj) acc[jj] = opfma<T, HERM>(kv[u][jj], xn, acc[jj]);
        }
        __syncthreads();
    }
    ts_finish_cols<T, HERM, CPW>(acc, c, 0, red, out, nullptr);
}

// xo = x - sum_j K[:, j] cin[j]  (thread per row, c read from shared memory)
template <class T>
__global__ void __launch_bounds__(256) ts_N(const T* __restrict__ K, long ldk, int c, const T* __restrict__ x,
                                            T* __restrict__ xo, long n, const double* __restrict__ cin,
                                            double csign, const CGState* st) {
    if (st && st->done) return;
    extern __shared__ double s_c[];
    constexpr int W = Sc<T>::W;
    for (int t = threadIdx.x; t < c * W; t += blockDim.x) s_c[t] = csign * cin[t];
    __syncthreads();
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += (long)gridDim.x * blockDim.x) {
        T acc = Sc<T>::zero();
        int j = 0;
        for (; j + 4 <= c; j += 4) {
            const T k0 = K[(size_t)j * ldk + row], k1 = K[(size_t)(j + 1) * ldk + row];
            const T k2 = K[(size_t)(j + 2) * ldk + row], k3 = K[(size_t)(j + 3) * ldk + row];
            acc = Sc<T>::fma(k0, Sc<T>::get(s_c + j * W), acc);
            acc = Sc<T>::fma(k1, Sc<T>::get(s_c + (j + 1) * W), acc);
            acc = Sc<T>::fma(k2, Sc<T>::get(s_c + (j + 2) * W), acc);
            acc = Sc<T>::fma(k3, Sc<T>::get(s_c + (j + 3) * W), acc);
        }
        for (; j < c; ++j) acc = Sc<T>::fma(K[(size_t)j * ldk + row], Sc<T>::get(s_c + j * W), acc);
        xo[row] = Sc<T>::sub(x[row], acc);
    }
}

// K4: q = w - K c2 ; p = r + beta p ; s = q + beta s ; y += alpha p ; r -= alpha s
template <class T, bool RB>
__global__ void __launch_bounds__(256) cg_update(const T* __restrict__ K, long ldk, int c, const T* __restrict__ w,
                                                 long n, const double* __restrict__ c2, T* __restrict__ r,
                                                 T* __restrict__ p, T* __restrict__ s, T* __restrict__ y,
                                                 CGState* st) {
    if (st->done) return;
    extern __shared__ double s_c[];
    constexpr int W = Sc<T>::W;
    for (int t = threadIdx.x; t < c * W; t += blockDim.x) s_c[t] = c2[t];
    __syncthreads();
    const T alpha = ld2<T>(st->alpha), beta = ld2<T>(st->beta);
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += (long)gridDim.x * blockDim.x) {
        T acc = Sc<T>::zero();
        int j = 0;
        for (; j + 8 <= c; j += 8) {
            T kk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) kk[q] = ldg_nc(K + kaddr<RB>(row, j + q, ldk));
#pragma unroll
            for (int q = 0; q < 8; ++q) reg_fence(kk[q]);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = Sc<T>::fma(kk[q], Sc<T>::get(s_c + (j + q) * W), acc);
        }
        for (; j < c; ++j) acc = Sc<T>::fma(K[kaddr<RB>(row, j, ldk)], Sc<T>::get(s_c + j * W), acc);
        const T q = Sc<T>::sub(w[row], acc);
        const T pn = Sc<T>::fma(beta, p[row], r[row]);
        const T sn = Sc<T>::fma(beta, s[row], q);
        p[row] = pn;
        s[row] = sn;
        y[row] = Sc<T>::fma(alpha, pn, y[row]);
        r[row] = Sc<T>::sub(r[row], Sc<T>::mul(alpha, sn));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->gamma_prev = st->gamma;
        st->alpha_prev = st->alpha;
        st->it = st->it + 1;
    }
}

// ------------------------------------------------------- vector utils ---
// out[0] = ||x||^2 (Hermitian), out[1..] = optional bilinear x^T x (complex)
template <class T>
__global__ void __launch_bounds__(256) vec_norms(const T* __restrict__ x, long n, GridRed red, double* out) {
    constexpr int W = Sc<T>::W;
    double h = 0.0;
    T b = Sc<T>::zero();
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const T v = x[i];
        h += Sc<T>::abs2(v);
        b = Sc<T>::fma(v, v, b);
    }
    __shared__ double s_red[32];
    __shared__ double s_vals[1 + W];
    double v[1 + W];
    v[0] = h;
    if constexpr (W == 1) {
        v[1] = b;
    } else {
        v[1] = ((cplx&)b).x;
        v[2] = ((cplx&)b).y;
    }
#pragma unroll
    for (int t = 0; t < 1 + W; ++t) {
        const double s = block_sum(v[t], s_red);
        if (threadIdx.x == 0) s_vals[t] = s;
    }
    __syncthreads();
    if (!grid_commit(red, s_vals, 1 + W)) return;
    grid_finish(red, 1 + W, out);
}

// ---- vector pieces of the reference's MINRES (krylov.cpp:17-98), real only ----
// The reference-faithful parity solver (ctx solver 1): Lanczos scalars live on
// the host, these kernels do the n-vector work. Rounded operation by operation
// like the reference's expressions (no FMA contraction).
// out[0] = a . b
__global__ void __launch_bounds__(256) vec_dot(const double* __restrict__ a, const double* __restrict__ b, long n,
                                               GridRed red, double* out) {
    double h = 0.0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        h = __dadd_rn(h, __dmul_rn(a[i], b[i]));
    __shared__ double s_red[32];
    __shared__ double s_vals[1];
    const double s = block_sum(h, s_red);
    if (threadIdx.x == 0) s_vals[0] = s;
    __syncthreads();
    if (!grid_commit(red, s_vals, 1)) return;
    grid_finish(red, 1, out);
}

// v = v / s (krylov.cpp:38: v = b / beta1)
__global__ void __launch_bounds__(256) vec_div(double* v, double s, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        v[i] = __ddiv_rn(v[i], s);
}

// p -= alpha v + beta v_old (krylov.cpp:52)
__global__ void __launch_bounds__(256) minres_lanczos(double* p, const double* __restrict__ v,
                                                      const double* __restrict__ v_old, double alpha, double beta,
                                                      long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        p[i] = __dsub_rn(p[i], __dadd_rn(__dmul_rn(alpha, v[i]), __dmul_rn(beta, v_old[i])));
}

// d_new = (v - delta d_old - eps d_oold) / gamma ; x += cphi d_new (krylov.cpp:64-65);
// then the rotation of krylov.cpp:87-91: v_old = v, v = p / beta_next (when
// advance), d_oold = d_old, d_old = d_new
__global__ void __launch_bounds__(256) minres_update(double* x, double* v, double* v_old, const double* __restrict__ p,
                                                     double* d_old, double* d_oold, double delta, double eps,
                                                     double gamma, double cphi, double beta_next, int advance, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const double vi = v[i], d1 = d_old[i], d2 = d_oold[i];
        const double dn = __ddiv_rn(__dsub_rn(__dsub_rn(vi, __dmul_rn(delta, d1)), __dmul_rn(eps, d2)), gamma);
        x[i] = __dadd_rn(x[i], __dmul_rn(cphi, dn));
        if (advance) {
            v_old[i] = vi;
            v[i] = __ddiv_rn(p[i], beta_next);
            d_oold[i] = d1;
            d_old[i] = dn;
        }
    }
}

// y = x * (1/rho) with rho from device: mode 0 = sqrt(out[0]) (Hermitian norm),
// mode 1 = complex sqrt of the bilinear x^T x (out[1], out[2]) (real: sqrt(out[1]))
template <class T> __device__ __forceinline__ T inv_rho(const double* nrm, int mode);
template <> __device__ __forceinline__ double inv_rho<double>(const double* nrm, int mode) {
    return 1.0 / sqrt(mode == 0 ? nrm[0] : nrm[1]);
}
template <> __device__ __forceinline__ cplx inv_rho<cplx>(const double* nrm, int mode) {
    if (mode == 0) return make_double2(1.0 / sqrt(nrm[0]), 0.0);
    // principal sqrt of a + ib
    const double a = nrm[1], b = nrm[2];
    const double m = sqrt(a * a + b * b);
    double sr = sqrt(0.5 * (m + a));
    double si = sqrt(fmax(0.0, 0.5 * (m - a)));
    if (b < 0) si = -si;
    return Sc<cplx>::div(make_double2(1.0, 0.0), make_double2(sr, si));
}

template <class T>
__global__ void vec_scale_by_rho(const T* __restrict__ x, T* __restrict__ y, long n, const double* nrm, int mode) {
    const T s = inv_rho<T>(nrm, mode);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        y[i] = Sc<T>::mul(x[i], s);
}

// y = a*x + y (a device scalar pair, optional) -- generic axpy with host scalar
template <class T>
__global__ void vec_axpby(long n, double2 a, const T* __restrict__ x, double2 b, T* __restrict__ y) {
    const T aa = ld2<T>(a), bb = ld2<T>(b);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        y[i] = Sc<T>::add(Sc<T>::mul(aa, x[i]), Sc<T>::mul(bb, y[i]));
}

// out[j] = op(K[idx, j]) * val   (row gather: K^op b for a single-nonzero b)
template <class T, bool HERM>
__global__ void row_gather(const T* __restrict__ K, long ldk, int c, long idx, double val, double* out) {
    constexpr int W = Sc<T>::W;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) {
        T k = K[(size_t)j * ldk + idx];
        T v = opmul<T, HERM>(k, Sc<T>::from(val));
        Sc<T>::put(out + (size_t)j * W, v);
    }
}

// out = a - b (device double arrays), or out = a + b
__global__ void dvec_addsub(int m, const double* a, const double* b, double sgn, double* out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) out[t] = a[t] + sgn * b[t];
}

// Seeded N(0,1) vector: splitmix64(seed, i) -> two uniforms -> Box-Muller.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__global__ void vec_randn(double* x, long n, uint64_t seed) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const uint64_t a = splitmix64(seed ^ (2 * (uint64_t)i)), b = splitmix64(seed ^ (2 * (uint64_t)i + 1));
        const double u1 = ((a >> 11) + 1.0) * 0x1.0p-53, u2 = ((b >> 11) + 1.0) * 0x1.0p-53;
        x[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

// Gershgorin bound max_p (|diag| + |shift| + sum |offdiag|) (krylov.cpp:190-195)
__global__ void __launch_bounds__(256) op_gershgorin(OpDev op, GridRed red, double* out) {
    double m = 0.0;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < op.n; p += (long)gridDim.x * blockDim.x) {
        int i, j, k;
        node_coords(op, p, i, j, k);
        // A applied to e_p gives column p = row p (symmetric); recompute the row sums directly
        const double Dp = op.D[p];
        double diag = op.mu[p], off = 0.0;
        const int idx[3] = {i, j, k};
        const int len[3] = {op.N0, op.N1, op.N2};
        const long st[3] = {1, op.N0, (long)op.N0 * op.N1};
        for (int ax = 0; ax < op.d; ++ax)
            for (int dir = -1; dir <= 1; dir += 2) {
                const int q = idx[ax] + dir;
                if (q >= 0 && q < len[ax]) {
                    const double f = hmean(Dp, op.D[p + dir * st[ax]]);
                    diag += f;
                    off += f;
                } else {
                    diag += (ax == op.d - 1) ? op.robin_face : Dp;
                }
            }
        m = fmax(m, fabs(diag) + fabs(op.shift) + off);
    }
    __shared__ double s_m[32];
    __shared__ double s_v[1];
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, s_m[w]);
        s_v[0] = b;
    }
    __syncthreads();
    if (!grid_commit(red, s_v, 1)) return;
    __threadfence();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (unsigned q = 0; q < gridDim.x * gridDim.y; ++q) b = fmax(b, __ldcg(red.partials + q));
        out[0] = b;
        *red.counter = 0u;
    }
}

// out[i + j*ldo] = sgn * op(K[idx[j], col0 + i]) * val[j]  (i < ncols, j < nrhs): the
// coordinates K^op b_j of single-nonzero right-hand sides, for many RHS at once.
template <class T, bool HERM>
__global__ void row_gather_multi(const T* __restrict__ K, long ldk, int col0, int ncols, const long* __restrict__ idx,
                                 const double* __restrict__ val, int nrhs, double sgn, T* __restrict__ out, long ldo) {
    const long tot = (long)ncols * nrhs;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e % ncols), j = (int)(e / ncols);
        const T k = K[(size_t)(col0 + i) * ldk + idx[j]];
        out[(size_t)j * ldo + i] = opmul<T, HERM>(k, Sc<T>::from(sgn * val[j]));
    }
}

// R[idx[j] + j*ldr] += val[j]
template <class T>
__global__ void scatter_add_rhs(T* R, long ldr, const long* __restrict__ idx, const double* __restrict__ val, int nrhs) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nrhs) {
        T& v = R[(size_t)j * ldr + idx[j]];
        v = Sc<T>::add(v, Sc<T>::from(val[j]));
    }
}

}  // namespace rd
