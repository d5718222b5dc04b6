// Batched recycled CG / COCG: M independent correction solves of ONE system in
// flight, each with its own recurrence (cg_recurrence, kernels.cuh), sharing the
// stream of the system's eigen block.
//
// Every recycle space of a system is K_j = [Kb | Kt_j]: the k leading columns
// (the factored eigen block, identical for every right-hand side of the system)
// and a few trailing columns of its own (X0_j and the corrections it appended).
// The one-solve iteration streams all of K_j twice per step (c1 = K_j^T A r,
// then q = A r - K_j c'); with M solves in flight the shared block is streamed
// once for all of them, so its bytes per solve-iteration fall by M:
//
//   stencil_tma   W[:, m] = A R[:, m]        all slots, coefficient planes read once
//   bd_dots       {r^T r, r^T w, r^H r}, alpha / beta / convergence per slot
//   bd_T_eig      C1e[m] = Kb^T W[:, m]      Kb: 1D bulk TMA ring, once for all m
//   bd_T_trail    C1t[m] = Kt_m^T W[:, m]
//   bd_coef       c'_m = 2 c1_m - G_m c1_m   (Gram-corrected second CGS coefficient)
//   bd_N_eig      W[:, m] -= Kb c'e_m        Kb streamed once for all m
//   bd_update     q = W[:, m] - Kt_m c't_m ; p = r + beta p ; s = q + beta s ;
//                 y += alpha p ; r -= alpha s ; it += 1
//
// Solves are only batched where the reference's loop (basis.cpp:168-205) leaves
// them independent: once the candidate cap stops the appends, no right-hand side
// changes the state another one starts from. A slot whose solve has finished
// (st[m].done) is skipped by every kernel: its W tile is not loaded, its
// accumulators are not touched. Each slot's arithmetic depends only on its own
// data and on the fixed row tiling, never on what the other slots hold, so a
// solve's result does not depend on the batch it ran in.
#pragma once

#include "dense.cuh"
#include "ts_tma.cuh"

namespace rd {

constexpr int BD_M = 16;      // slots in flight (two 8-slot DMMA column groups)
constexpr int BD_TCH = 8;     // trailing columns per bd_T_trail chunk
constexpr int BD_NCH = 3;     // chunks: trailing width <= 24

template <class T> struct BDTrail {  // trailing blocks of the slots (column-major, ld rows apart)
    const T* Kt[BD_M];
    int t[BD_M];
};

struct BDLayout {
    int TR, S, kb;
    uint32_t tile_bytes, x_bytes, stride_k, stride_x;
    uint32_t off_k, off_x, off_vals, off_bar, total;
    uint32_t cstride;  // N pass: elements between the slots' coefficient rows in shared memory
};

// TR rows per tile; xpad bytes between the slots' W tiles (bank spread of the
// fragment loads: 64 for the T pass, 16 for the N pass).
template <class T> inline BDLayout bd_layout(int kb, int TR, int S, uint32_t xpad) {
    BDLayout L;
    L.kb = kb;
    L.TR = TR;
    L.S = S;
    L.tile_bytes = (uint32_t)TR * kb * sizeof(T);
    L.x_bytes = (uint32_t)TR * sizeof(T);
    auto al = [](uint32_t v) { return (v + 127u) & ~127u; };
    L.stride_k = al(L.tile_bytes);
    L.stride_x = L.x_bytes + xpad;
    uint32_t o = 0;
    L.off_k = o;
    o += L.stride_k * S;
    L.off_x = o;
    o += al(L.stride_x * BD_M) * S;
    L.off_vals = o;  // T pass: the block's M kb partial sums; N pass: the coefficients (padded rows)
    // N pass rows cover every column the unrolled DMMA steps touch (4, 8 or 16 steps of 4)
    L.cstride = (kb <= 16 ? 16u : kb <= 32 ? 32u : 64u) + 4u;
    o += al((uint32_t)BD_M * L.cstride * 2 * sizeof(double));
    L.off_bar = o;
    o += 2 * S * 8;
    L.total = o;
    return L;
}

// The eigen block in 4-row blocks: element (row, col) of the n x kb block sits at
// (row / 4) (4 kb) + 4 col + row % 4, so TR consecutive rows are one contiguous
// chunk (one bulk TMA copy) and the 8 x 4 DMMA fragment of K^T (8 columns x 4
// rows) is 32 consecutive elements.
template <class T>
__global__ void repack_q4(const T* __restrict__ K, long ldk, int kb, long n, T* __restrict__ out, long nrows_out) {
    const long tot = nrows_out * (long)kb;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
        const long q = e / (4L * kb);
        const int rem = (int)(e - q * 4L * kb);
        const int j = rem >> 2;
        const long row = q * 4 + (rem & 3);
        out[e] = row < n ? K[(size_t)j * ldk + row] : Sc<T>::zero();
    }
}

// acc (8 x 8 tile, C fragment: row lane/4, columns 2 (lane%4) + {0, 1}) += A B
// for one k-step of 4; complex as four real DMMA (bilinear product).
template <class T> struct BDAcc;
template <> struct BDAcc<double> {
    double r0 = 0.0, r1 = 0.0;
    __device__ __forceinline__ void mma(double a, double b) { dmma(r0, r1, a, b); }
    __device__ __forceinline__ double get(int e) const { return e ? r1 : r0; }
};
template <> struct BDAcc<cplx> {
    double r0 = 0.0, r1 = 0.0, i0 = 0.0, i1 = 0.0;
    __device__ __forceinline__ void mma(cplx a, cplx b) {
        dmma(r0, r1, a.x, b.x);
        dmma(r0, r1, -a.y, b.y);
        dmma(i0, i1, a.x, b.y);
        dmma(i0, i1, a.y, b.x);
    }
    __device__ __forceinline__ cplx get(int e) const { return e ? make_double2(r1, i1) : make_double2(r0, i0); }
};

// C1e[m][0..kb) = Kb^T W[:, m] for every running slot, on the FP64 tensor
// cores: warp w owns columns [8w, 8w + 8) of Kb; per 4 rows one DMMA step with
// A = K^T (8 columns x 4 rows) and B = W (4 rows x 8 slots); the 8 x 8
// accumulator tile lives in 2 (real) / 4 (complex) registers per lane. One
// deterministic grid reduction of M kb values.
template <class T>
__global__ void __launch_bounds__(TMA_THREADS, 1)
    bd_T_eig(const T* __restrict__ Kq, long n, long ntile, BDLayout L, const T* __restrict__ Wv, long ld,
             const CGState* __restrict__ st, GridRed red, double* __restrict__ out) {
    constexpr int W = Sc<T>::W;
    constexpr int M = BD_M;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned s_act;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int kb = L.kb, TR = L.TR, S = L.S;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
    uint64_t* empty = full + S;
    double* vals = reinterpret_cast<double*>(smem + L.off_vals);
    const uint32_t xstage = (L.stride_x * M + 127u) & ~127u;
    if (tid == 0) {
        unsigned a = 0;
        for (int m = 0; m < M; ++m) a |= (st[m].done ? 0u : 1u) << m;
        s_act = a;
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], TMA_CONSUMERS / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned act = s_act;
    if (!act) return;
    const int nact = __popc(act);
    if (wid == TMA_CONSUMERS / 32) {
        if (lane == 0) {
            long k = 0;
            for (long t = blockIdx.x; t < ntile; t += gridDim.x, ++k) {
                const int stage = (int)(k % S);
                const uint32_t use = (uint32_t)(k / S);
                mbar_wait(&empty[stage], (use & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[stage], L.tile_bytes + nact * L.x_bytes);
                tma_load_1d(smem + L.off_k + stage * L.stride_k, Kq + (size_t)t * TR * kb, L.tile_bytes, &full[stage]);
                unsigned char* xb = smem + L.off_x + (size_t)stage * xstage;
                for (int m = 0; m < M; ++m)
                    if (act >> m & 1u)
                        tma_load_1d(xb + m * L.stride_x, Wv + (size_t)m * ld + (size_t)t * TR, L.x_bytes, &full[stage]);
            }
        }
    } else {
        const int fi = lane >> 2, fk = lane & 3;
        const int j0 = wid * 8;
        const bool warp_on = j0 < kb;
        const bool colok = j0 + fi < kb;
        // B fragment columns = slots fi and 8 + fi (two 8-slot groups share the A fragment)
        const bool bact0 = act >> fi & 1u, bact1 = act >> (8 + fi) & 1u;
        const bool hi = (act >> 8) != 0u;
        BDAcc<T> acc0, acc1;
        const int nstep = TR >> 2;
        long k = 0;
        for (long t = blockIdx.x; t < ntile; t += gridDim.x, ++k) {
            const int stage = (int)(k % S);
            const uint32_t use = (uint32_t)(k / S);
            mbar_wait(&full[stage], use & 1u);
            if (warp_on) {
                const T* ks = reinterpret_cast<const T*>(smem + L.off_k + stage * L.stride_k) + (j0 + fi) * 4 + fk;
                const unsigned char* xb = smem + L.off_x + (size_t)stage * xstage;
                const T* xs0 = reinterpret_cast<const T*>(xb + fi * L.stride_x) + fk;
                const T* xs1 = reinterpret_cast<const T*>(xb + (8 + fi) * L.stride_x) + fk;
                if (hi) {
#pragma unroll 4
                    for (int s = 0; s < nstep; ++s) {
                        const T a = colok ? ks[(size_t)s * 4 * kb] : Sc<T>::zero();
                        const T b0 = bact0 ? xs0[4 * s] : Sc<T>::zero();
                        const T b1 = bact1 ? xs1[4 * s] : Sc<T>::zero();
                        acc0.mma(a, b0);
                        acc1.mma(a, b1);
                    }
                } else {
#pragma unroll 8
                    for (int s = 0; s < nstep; ++s) {
                        const T a = colok ? ks[(size_t)s * 4 * kb] : Sc<T>::zero();
                        const T b0 = bact0 ? xs0[4 * s] : Sc<T>::zero();
                        acc0.mma(a, b0);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
        }
        if (colok) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int m = 2 * fk + e;
                Sc<T>::put(vals + ((size_t)m * kb + j0 + fi) * W, acc0.get(e));
                Sc<T>::put(vals + ((size_t)(8 + m) * kb + j0 + fi) * W, acc1.get(e));
            }
        }
    }
    __syncthreads();
    if (!grid_commit(red, vals, M * kb * W)) return;
    grid_finish(red, M * kb * W, out);
}

// W[:, m] -= Kb c'e_m for every running slot (in place), on the FP64 tensor
// cores: a warp owns 8 rows of the tile at a time; A = K (8 rows x 4 columns
// per step), B = the coefficients (4 columns x 8 slots, held in registers for
// the whole launch). No cross-warp reduction.
template <class T, int NSTEP>
__global__ void __launch_bounds__(TMA_THREADS, 1)
    bd_N_eig(const T* __restrict__ Kq, long n, long ntile, BDLayout L, T* __restrict__ Wv, long ld,
             const CGState* __restrict__ st, const double* __restrict__ cpe) {
    constexpr int W = Sc<T>::W;
    constexpr int M = BD_M;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned s_act;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int kb = L.kb, TR = L.TR, S = L.S;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
    uint64_t* empty = full + S;
    const uint32_t xstage = (L.stride_x * M + 127u) & ~127u;
    if (tid == 0) {
        unsigned a = 0;
        for (int m = 0; m < M; ++m) a |= (st[m].done ? 0u : 1u) << m;
        s_act = a;
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], TMA_CONSUMERS / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned act = s_act;
    if (!act) return;
    const int nact = __popc(act);
    // coefficient rows of all slots (zero for finished slots and padded columns)
    T* cs = reinterpret_cast<T*>(smem + L.off_vals);
    for (int e = tid; e < M * (int)L.cstride; e += blockDim.x) {
        const int m = e / (int)L.cstride, col = e - m * (int)L.cstride;
        cs[e] = (col < kb && (act >> m & 1u)) ? Sc<T>::get(cpe + ((size_t)m * kb + col) * W) : Sc<T>::zero();
    }
    __syncthreads();
    if (wid == TMA_CONSUMERS / 32) {
        if (lane == 0) {
            long k = 0;
            for (long t = blockIdx.x; t < ntile; t += gridDim.x, ++k) {
                const int stage = (int)(k % S);
                const uint32_t use = (uint32_t)(k / S);
                mbar_wait(&empty[stage], (use & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[stage], L.tile_bytes + nact * L.x_bytes);
                tma_load_1d(smem + L.off_k + stage * L.stride_k, Kq + (size_t)t * TR * kb, L.tile_bytes, &full[stage]);
                unsigned char* xb = smem + L.off_x + (size_t)stage * xstage;
                for (int m = 0; m < M; ++m)
                    if (act >> m & 1u)
                        tma_load_1d(xb + m * L.stride_x, Wv + (size_t)m * ld + (size_t)t * TR, L.x_bytes, &full[stage]);
            }
        }
        return;
    }
    const int fi = lane >> 2, fk = lane & 3;
    const bool hi = (act >> 8) != 0u;
    // B fragments (coefficient of column 4 s + fk for slots fi and 8 + fi) are read from the
    // staged coefficient rows at every step: 2 x NSTEP register copies would not fit
    const T* cf0 = cs + (size_t)fi * L.cstride + fk;
    const T* cf1 = cs + (size_t)(8 + fi) * L.cstride + fk;
    const int ngroup = TR >> 3;
    long k = 0;
    for (long t = blockIdx.x; t < ntile; t += gridDim.x, ++k) {
        const int stage = (int)(k % S);
        const uint32_t use = (uint32_t)(k / S);
        mbar_wait(&full[stage], use & 1u);
        const T* Ks = reinterpret_cast<const T*>(smem + L.off_k + stage * L.stride_k);
        const unsigned char* xb = smem + L.off_x + (size_t)stage * xstage;
        for (int g = wid; g < ngroup; g += TMA_CONSUMERS / 32) {
            const int r = 8 * g + fi;
            const T* ks = Ks + (size_t)(r >> 2) * 4 * kb + (r & 3) + 4 * fk;
            BDAcc<T> acc0, acc1;
            if (hi) {
#pragma unroll
                for (int s = 0; s < NSTEP; ++s) {
                    const T a = (4 * s + fk < kb) ? ks[16 * s] : Sc<T>::zero();
                    acc0.mma(a, cf0[4 * s]);
                    acc1.mma(a, cf1[4 * s]);
                }
            } else {
#pragma unroll
                for (int s = 0; s < NSTEP; ++s) {
                    const T a = (4 * s + fk < kb) ? ks[16 * s] : Sc<T>::zero();
                    acc0.mma(a, cf0[4 * s]);
                }
            }
            const long row = t * TR + r;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = 8 * h + 2 * fk + e;
                    if ((act >> m & 1u) && row < n) {
                        const T wv = reinterpret_cast<const T*>(xb + m * L.stride_x)[r];
                        Wv[(size_t)m * ld + row] = Sc<T>::sub(wv, h ? acc1.get(e) : acc0.get(e));
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
}

// Merged reduction {r^T r, r^T w, r^H r} of every running slot (blockIdx.y) and,
// in the slot's last block, its scalar recurrence step (alpha, beta, convergence:
// cg_recurrence). w = A r comes from the multi-column TMA stencil, which reads the
// coefficient planes once for all slots.
template <class T>
__global__ void __launch_bounds__(256, 4) bd_dots(const T* __restrict__ R, const T* __restrict__ Wv, long ld, long n,
                                                  CGState* st, double* partials, unsigned* counters,
                                                  double* hist0 /* [slot]: relres of iteration 0, or null */) {
    constexpr int W = Sc<T>::W;
    constexpr int NV = 2 * W + 1;
    const int m = blockIdx.y;
    CGState* sc = st + m;
    if (sc->done) return;
    const T* __restrict__ r = R + (size_t)m * ld;
    const T* __restrict__ w = Wv + (size_t)m * ld;
    T g = Sc<T>::zero(), dl = Sc<T>::zero();
    double h = 0.0;
    const long stride = (long)gridDim.x * blockDim.x;
    long row = blockIdx.x * (long)blockDim.x + threadIdx.x;
    for (; row + stride < n; row += 2 * stride) {
        const T r0 = r[row], w0 = w[row], r1 = r[row + stride], w1 = w[row + stride];
        g = Sc<T>::fma(r0, r0, g);
        dl = Sc<T>::fma(r0, w0, dl);
        h += Sc<T>::abs2(r0);
        g = Sc<T>::fma(r1, r1, g);
        dl = Sc<T>::fma(r1, w1, dl);
        h += Sc<T>::abs2(r1);
    }
    if (row < n) {
        const T r0 = r[row], w0 = w[row];
        g = Sc<T>::fma(r0, r0, g);
        dl = Sc<T>::fma(r0, w0, dl);
        h += Sc<T>::abs2(r0);
    }
    __shared__ double s_red[32];
    __shared__ double s_vals[NV];
    double v[NV];
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
    for (int t = 0; t < NV; ++t) {
        const double sv = block_sum(v[t], s_red);
        if (threadIdx.x == 0) s_vals[t] = sv;
    }
    __syncthreads();
    GridRed red{partials + (size_t)m * gridDim.x * NV, counters + m};
    if (!grid_commit_at(red, s_vals, NV, blockIdx.x, gridDim.x)) return;
    __shared__ double s_tot[NV];
    grid_finish(red, NV, s_tot, gridDim.x);
    if (threadIdx.x != 0) return;
    cg_recurrence<T>(sc, s_tot, hist0 ? hist0 + m : nullptr);  // hist_cap = 1: only iteration 0 is recorded
}

// Partial dots of TW trailing columns against w over this block's rows: one
// row per thread and trip, its 1 + TW loads issued before the first FMA (a
// double2 is four registers: wider per-thread batches cost occupancy, and the
// pass needs resident warps more than it needs loads per warp).
template <class T, int TW>
__device__ __forceinline__ void bd_trail_dots(const T* __restrict__ Kt, long ld, const T* __restrict__ w, long n,
                                              T (&acc)[BD_TCH]) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += stride) {
        const T wv = w[row];
        T kv[TW];
#pragma unroll
        for (int q = 0; q < TW; ++q) kv[q] = Kt[(size_t)q * ld + row];
#pragma unroll
        for (int q = 0; q < TW; ++q) acc[q] = Sc<T>::fma(kv[q], wv, acc[q]);
    }
}

// C1t[m][0..t_m) = Kt_m^T W[:, m]: blockIdx.y = slot, thread per row, chunks of
// BD_TCH columns; per (slot, chunk) deterministic reduction over the blocks.
template <class T>
__global__ void __launch_bounds__(256, 4) bd_T_trail(BDTrail<T> tr, const T* __restrict__ Wv, long ld, long n,
                                                  const CGState* __restrict__ st, double* partials,
                                                  unsigned* counters, double* __restrict__ out, int tcap) {
    constexpr int W = Sc<T>::W;
    const int m = blockIdx.y;
    if (st[m].done) return;
    const int t = tr.t[m];
    const T* __restrict__ w = Wv + (size_t)m * ld;
    __shared__ double s_red[32];
    __shared__ double s_vals[BD_TCH * W];
    for (int ch = 0, t0 = 0; t0 < t; ++ch, t0 += BD_TCH) {
        const T* __restrict__ Kt = tr.Kt[m] + (size_t)t0 * ld;
        T acc[BD_TCH];
#pragma unroll
        for (int q = 0; q < BD_TCH; ++q) acc[q] = Sc<T>::zero();
        switch (min(t - t0, BD_TCH)) {
            case 1: bd_trail_dots<T, 1>(Kt, ld, w, n, acc); break;
            case 2: bd_trail_dots<T, 2>(Kt, ld, w, n, acc); break;
            case 3: bd_trail_dots<T, 3>(Kt, ld, w, n, acc); break;
            case 4: bd_trail_dots<T, 4>(Kt, ld, w, n, acc); break;
            case 5: bd_trail_dots<T, 5>(Kt, ld, w, n, acc); break;
            case 6: bd_trail_dots<T, 6>(Kt, ld, w, n, acc); break;
            case 7: bd_trail_dots<T, 7>(Kt, ld, w, n, acc); break;
            default: bd_trail_dots<T, 8>(Kt, ld, w, n, acc); break;
        }
#pragma unroll
        for (int q = 0; q < BD_TCH; ++q) {
            double a[W];
            if constexpr (W == 1) {
                a[0] = (double&)acc[q];
            } else {
                a[0] = ((cplx&)acc[q]).x;
                a[1] = ((cplx&)acc[q]).y;
            }
#pragma unroll
            for (int e = 0; e < W; ++e) {
                const double v = block_sum(a[e], s_red);
                if (threadIdx.x == 0) s_vals[q * W + e] = v;
            }
        }
        __syncthreads();
        const int slot = m * BD_NCH + ch;
        GridRed red{partials + (size_t)slot * gridDim.x * BD_TCH * W, counters + slot};
        if (grid_commit_at(red, s_vals, BD_TCH * W, blockIdx.x, gridDim.x))
            grid_finish(red, BD_TCH * W, out + ((size_t)m * tcap + t0) * W, gridDim.x);
        __syncthreads();
    }
}

// c'_m = 2 c1_m - G_m c1_m with c1_m = [C1e[m] ; C1t[m]] and G_m = K_m^T K_m
// (cj x cj, symmetric). One block per slot.
template <class T>
__global__ void __launch_bounds__(128) bd_coef(BDTrail<T> tr, int kb, int tcap, const CGState* __restrict__ st,
                                               const double* __restrict__ c1e, const double* __restrict__ c1t,
                                               const T* __restrict__ G, long gstride, double* __restrict__ cpe,
                                               double* __restrict__ cpt) {
    constexpr int W = Sc<T>::W;
    const int m = blockIdx.x;
    if (st[m].done) return;
    const int cj = kb + tr.t[m];
    extern __shared__ __align__(16) unsigned char sm_[];
    T* c1 = reinterpret_cast<T*>(sm_);
    for (int j = threadIdx.x; j < cj; j += blockDim.x)
        c1[j] = j < kb ? Sc<T>::get(c1e + ((size_t)m * kb + j) * W) : Sc<T>::get(c1t + ((size_t)m * tcap + j - kb) * W);
    __syncthreads();
    const T* Gm = G + (size_t)m * gstride;
    for (int j = threadIdx.x; j < cj; j += blockDim.x) {
        // G is symmetric: walk column j (consecutive threads read consecutive addresses)
        T a0 = Sc<T>::zero(), a1 = Sc<T>::zero(), a2 = Sc<T>::zero(), a3 = Sc<T>::zero();
        int i = 0;
        for (; i + 3 < cj; i += 4) {
            a0 = Sc<T>::fma(Gm[(size_t)i * cj + j], c1[i], a0);
            a1 = Sc<T>::fma(Gm[(size_t)(i + 1) * cj + j], c1[i + 1], a1);
            a2 = Sc<T>::fma(Gm[(size_t)(i + 2) * cj + j], c1[i + 2], a2);
            a3 = Sc<T>::fma(Gm[(size_t)(i + 3) * cj + j], c1[i + 3], a3);
        }
        for (; i < cj; ++i) a0 = Sc<T>::fma(Gm[(size_t)i * cj + j], c1[i], a0);
        const T acc = Sc<T>::add(Sc<T>::add(a0, a1), Sc<T>::add(a2, a3));
        const T v = Sc<T>::sub(Sc<T>::scale(c1[j], 2.0), acc);
        if (j < kb)
            Sc<T>::put(cpe + ((size_t)m * kb + j) * W, v);
        else
            Sc<T>::put(cpt + ((size_t)m * tcap + j - kb) * W, v);
    }
}

// Rows of one trip of bd_update with a compile-time trailing width (all loads
// of the trip issued up front).
template <class T, int TW>
__device__ __forceinline__ T bd_trail_row(const T* __restrict__ Kt, long ld, long row, const T* s_c) {
    T kv[TW > 0 ? TW : 1];
#pragma unroll
    for (int q = 0; q < TW; ++q) kv[q] = Kt[(size_t)q * ld + row];
    T sum = Sc<T>::zero();
#pragma unroll
    for (int q = 0; q < TW; ++q) sum = Sc<T>::fma(kv[q], s_c[q], sum);
    return sum;
}

// q = W[:, m] - Kt_m c't_m, then the CG / COCG vector updates of slot m
// (blockIdx.y), thread per row; block 0 advances the slot's iteration count.
template <class T>
__global__ void __launch_bounds__(256) bd_update(BDTrail<T> tr, const T* __restrict__ Wv, T* __restrict__ R,
                                                 T* __restrict__ Pv, T* __restrict__ Sv, T* __restrict__ Y, long ld,
                                                 long n, CGState* st, const double* __restrict__ cpt, int tcap) {
    constexpr int W = Sc<T>::W;
    const int m = blockIdx.y;
    CGState* sc = st + m;
    if (sc->done) return;
    const int t = tr.t[m];
    const T* __restrict__ Kt = tr.Kt[m];
    __shared__ T s_c[BD_TCH * BD_NCH];
    if (threadIdx.x < t) s_c[threadIdx.x] = Sc<T>::get(cpt + ((size_t)m * tcap + threadIdx.x) * W);
    __syncthreads();
    const T alpha = ld2<T>(sc->alpha), beta = ld2<T>(sc->beta);
    const size_t off = (size_t)m * ld;
    for (long row = blockIdx.x * (long)blockDim.x + threadIdx.x; row < n; row += (long)gridDim.x * blockDim.x) {
        const T wv = Wv[off + row], rv = R[off + row], pv = Pv[off + row], sv = Sv[off + row], yv = Y[off + row];
        T sum = Sc<T>::zero();
        int t0 = 0;
        for (; t0 + 8 <= t; t0 += 8) sum = Sc<T>::add(sum, bd_trail_row<T, 8>(Kt + (size_t)t0 * ld, ld, row, s_c + t0));
        switch (t - t0) {
            case 1: sum = Sc<T>::add(sum, bd_trail_row<T, 1>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            case 2: sum = Sc<T>::add(sum, bd_trail_row<T, 2>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            case 3: sum = Sc<T>::add(sum, bd_trail_row<T, 3>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            case 4: sum = Sc<T>::add(sum, bd_trail_row<T, 4>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            case 5: sum = Sc<T>::add(sum, bd_trail_row<T, 5>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            case 6: sum = Sc<T>::add(sum, bd_trail_row<T, 6>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            case 7: sum = Sc<T>::add(sum, bd_trail_row<T, 7>(Kt + (size_t)t0 * ld, ld, row, s_c + t0)); break;
            default: break;
        }
        const T q = Sc<T>::sub(wv, sum);
        const T pn = Sc<T>::fma(beta, pv, rv);
        const T sn = Sc<T>::fma(beta, sv, q);
        Pv[off + row] = pn;
        Sv[off + row] = sn;
        Y[off + row] = Sc<T>::fma(alpha, pn, yv);
        R[off + row] = Sc<T>::sub(rv, Sc<T>::mul(alpha, sn));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->gamma_prev = sc->gamma;
        sc->alpha_prev = sc->alpha;
        sc->it = sc->it + 1;
    }
}

}  // namespace rd
