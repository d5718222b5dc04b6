// TMA-pipelined recycle-space projection kernels for the inner iteration.
//
// The per-RHS recycle basis K (n x C) is kept in the row-blocked layout
// (kaddr<true>), so a tile of TR consecutive rows x all C columns is ONE
// contiguous chunk of TR*C elements. A persistent CTA per SM runs a producer
// warp that streams tiles with 1D bulk TMA copies (cp.async.bulk + mbarrier
// complete_tx) into an S-stage shared-memory ring (~160 KB in flight per SM,
// what HBM3e needs at ~3 us loaded latency), and 8 consumer warps that compute
// from shared memory:
//
//   MODE 0  c   = op(K)^T x                          (first CGS pass)
//   MODE 1  x'  = x - K c1 ; c2 = op(K)^T x'         (fused second CGS pass)
//   MODE 2  q   = w' - K c2 ; p = r + beta p ; s = q + beta s ;
//           y  += alpha p ; r -= alpha s             (CG/COCG update)
//           with G = K^T K given: q = w - K (2 c1 - G c1), the one-pass
//           projection with the Gram-corrected second CGS coefficient
//   MODE 3  x'  = x - K c                            (N pass, global basis)
//
// TMAP = true streams a column-major matrix (the global basis V/W/K_img,
// ld = n) through a 2D tensor map instead: one cp.async.bulk.tensor.2d per
// 32-row x C-column box lands in shared memory in the same (column, 32-row)
// order as a row-blocked tile, so the consumers are shared; rows >= n are
// zero-filled by the TMA unit.
//
// Rows >= n are zero padding of K and of the x workspace. Reductions are the
// deterministic per-block partial + last-block sum of common.cuh.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "kernels.cuh"

namespace rd {

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

constexpr int TMA_CONSUMERS = 256;  // 8 warps
constexpr int TMA_THREADS = TMA_CONSUMERS + 32;

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

struct TmaLayout {
    int TR, S, NV;
    uint32_t tile_bytes, x_bytes;
    uint32_t off_k, off_x, off_part, off_xs, off_cw, off_vals, off_bar, total;
};

template <class T> __host__ __device__ inline TmaLayout tma_layout(int C, int TR, int S, int NV) {
    TmaLayout L;
    L.TR = TR;
    L.S = S;
    L.NV = NV;
    const uint32_t es = sizeof(T);
    L.tile_bytes = (uint32_t)TR * C * es;
    L.x_bytes = (uint32_t)TR * es;
    auto al = [](uint32_t v) { return (v + 127u) & ~127u; };
    uint32_t o = 0;
    L.off_k = o;
    o += al(L.tile_bytes) * S;
    L.off_x = o;
    o += al(L.x_bytes) * S * NV;
    L.off_part = o;
    o += al((uint32_t)2 * (TR / 32) * 8 * 32 * es);
    L.off_xs = o;
    o += al((uint32_t)TR * es);
    L.off_cw = o;
    o += al((uint32_t)(C > 0 ? C : 1) * es);
    L.off_vals = o;
    o += al((uint32_t)(C > 0 ? C : 1) * 2 * sizeof(double));
    L.off_bar = o;
    o += 2 * S * 8;
    L.total = o;
    return L;
}

template <class T, int MODE, bool HERM, int CPW, bool TMAP>
__global__ void __launch_bounds__(TMA_THREADS, 1)
    ts_tma(const __grid_constant__ CUtensorMap tmap, int col0, const T* __restrict__ Krb, int C, long n, long ntile,
           TmaLayout L, const T* __restrict__ x,
           T* __restrict__ xo, const double* __restrict__ cin, GridRed red, double* out, T* __restrict__ r,
           T* __restrict__ p, T* __restrict__ s, T* __restrict__ y, CGState* st, const T* __restrict__ G) {
    if (st && st->done) return;
    constexpr int W = Sc<T>::W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int TR = L.TR, S = L.S;
    const uint32_t stride_k = (L.tile_bytes + 127u) & ~127u;
    const uint32_t stride_x = (L.x_bytes + 127u) & ~127u;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
    uint64_t* empty = full + S;
    T* part = reinterpret_cast<T*>(smem + L.off_part);
    T* cw = reinterpret_cast<T*>(smem + L.off_cw);
    double* vals = reinterpret_cast<double*>(smem + L.off_vals);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], TMA_CONSUMERS / 32);
        }
        fence_mbar_init();
    }
    if (MODE == 2 && G) {
        // one-pass projection with the Gram correction: coef = c1 + (c1 - G c1),
        // the second CGS coefficient K^T (w - K c1) = c1 - (K^T K) c1 formed from
        // the solve's fixed Gram G = K^T K (symmetric: column t = row t) instead
        // of a third stream over K. c1 is staged in the vals region (unused here).
        T* c1s = reinterpret_cast<T*>(smem + L.off_vals);
        for (int t = tid; t < C; t += blockDim.x) c1s[t] = Sc<T>::get(cin + (size_t)t * W);
        __syncthreads();
        for (int t = tid; t < C; t += blockDim.x) {
            const T* gc = G + (size_t)t * C;
            T acc = Sc<T>::zero();
            for (int j = 0; j < C; ++j) acc = Sc<T>::fma(gc[j], c1s[j], acc);
            cw[t] = Sc<T>::sub(Sc<T>::scale(c1s[t], 2.0), acc);
        }
    } else if (MODE != 0) {
        for (int t = tid; t < C; t += blockDim.x) cw[t] = Sc<T>::get(cin + (size_t)t * W);
    }
    __syncthreads();

    if (wid == TMA_CONSUMERS / 32) {
        // ---------------- producer warp: one elected lane streams tiles ----------------
        if (lane == 0) {
            long k = 0;
            for (long t = blockIdx.x; t < ntile; t += gridDim.x, ++k) {
                const int stage = (int)(k % S);
                const uint32_t use = (uint32_t)(k / S);
                mbar_wait(&empty[stage], (use & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[stage], L.tile_bytes + L.NV * L.x_bytes);
                if constexpr (TMAP)
                    tma_load_2d(smem + L.off_k + stage * stride_k, &tmap, (int)(t * TR * Sc<T>::W), col0, &full[stage]);
                else
                    tma_load_1d(smem + L.off_k + stage * stride_k, Krb + (size_t)t * TR * C, L.tile_bytes,
                                &full[stage]);
                unsigned char* xb = smem + L.off_x + (size_t)stage * L.NV * stride_x;
                tma_load_1d(xb, x + (size_t)t * TR, L.x_bytes, &full[stage]);
                if (MODE == 2) {
                    tma_load_1d(xb + 1 * stride_x, r + (size_t)t * TR, L.x_bytes, &full[stage]);
                    tma_load_1d(xb + 2 * stride_x, p + (size_t)t * TR, L.x_bytes, &full[stage]);
                    tma_load_1d(xb + 3 * stride_x, s + (size_t)t * TR, L.x_bytes, &full[stage]);
                    tma_load_1d(xb + 4 * stride_x, y + (size_t)t * TR, L.x_bytes, &full[stage]);
                }
            }
        }
    } else {
        // ---------------- consumer warps ----------------
        const int j0 = wid * CPW;
        int ncol = C - j0;
        if (ncol > CPW) ncol = CPW;
        T acc[CPW];
#pragma unroll
        for (int jj = 0; jj < CPW; ++jj) acc[jj] = Sc<T>::zero();
        T alpha = Sc<T>::zero(), beta = Sc<T>::zero();
        if (MODE == 2) {
            alpha = ld2<T>(st->alpha);
            beta = ld2<T>(st->beta);
        }
        long k = 0;
        for (long t = blockIdx.x; t < ntile; t += gridDim.x, ++k) {
            const int stage = (int)(k % S);
            const uint32_t use = (uint32_t)(k / S);
            mbar_wait(&full[stage], use & 1u);
            const T* Ks = reinterpret_cast<const T*>(smem + L.off_k + stage * stride_k);
            const unsigned char* xb = smem + L.off_x + (size_t)stage * L.NV * stride_x;
            const T* Xs = reinterpret_cast<const T*>(xb);
            const long row0 = t * TR;
            const int RBN = TR >> 5;
            if (MODE == 0) {
                // T part: warp w owns columns [j0, j0 + CPW), lanes over the TR rows
                for (int rb = 0; rb < RBN; ++rb) {
                    const T xv = Xs[rb * 32 + lane];
                    const T* kb = Ks + (size_t)rb * 32 * C + lane;
#pragma unroll
                    for (int jj = 0; jj < CPW; ++jj)
                        if (jj < ncol) acc[jj] = opfma<T, HERM>(kb[(size_t)(j0 + jj) * 32], xv, acc[jj]);
                }
            } else {
                // N part on the same (column-block x lane) mapping: every warp forms the
                // partial row sums of its own columns; one barrier per tile (the partial
                // buffer alternates with the tile parity).
                T* pb = part + (size_t)(k & 1) * RBN * 8 * 32;
                for (int rb = 0; rb < RBN; ++rb) {
                    const T* kb = Ks + (size_t)rb * 32 * C + lane;
                    T pa = Sc<T>::zero();
#pragma unroll
                    for (int jj = 0; jj < CPW; ++jj)
                        if (jj < ncol) pa = Sc<T>::fma(kb[(size_t)(j0 + jj) * 32], cw[j0 + jj], pa);
                    pb[(rb * 8 + wid) * 32 + lane] = pa;
                }
                consumer_sync();
                if (MODE == 1) {
                    // the owner warp of each 32-row block reduces the 8 partial sums once
                    // into the shared q tile; a second barrier publishes it to every warp
                    // (reading all partials in every warp costs 8x the smem traffic)
                    T* qs = reinterpret_cast<T*>(smem + L.off_xs);
                    for (int rb = wid; rb < RBN; rb += 8) {
                        T sum = pb[(rb * 8) * 32 + lane];
#pragma unroll
                        for (int w2 = 1; w2 < 8; ++w2) sum = Sc<T>::add(sum, pb[(rb * 8 + w2) * 32 + lane]);
                        const long row = row0 + rb * 32 + lane;
                        T q = Sc<T>::sub(Xs[rb * 32 + lane], sum);
                        if (row >= n) q = Sc<T>::zero();
                        else xo[row] = q;
                        qs[rb * 32 + lane] = q;
                    }
                    consumer_sync();
                    for (int rb = 0; rb < RBN; ++rb) {
                        const T q = qs[rb * 32 + lane];
                        const T* kb = Ks + (size_t)rb * 32 * C + lane;
#pragma unroll
                        for (int jj = 0; jj < CPW; ++jj)
                            if (jj < ncol) acc[jj] = opfma<T, HERM>(kb[(size_t)(j0 + jj) * 32], q, acc[jj]);
                    }
                } else if (MODE == 3) {
                    for (int rb = wid; rb < RBN; rb += 8) {
                        T sum = pb[(rb * 8) * 32 + lane];
#pragma unroll
                        for (int w2 = 1; w2 < 8; ++w2) sum = Sc<T>::add(sum, pb[(rb * 8 + w2) * 32 + lane]);
                        const int rr = rb * 32 + lane;
                        const long row = row0 + rr;
                        if (row < n) xo[row] = Sc<T>::sub(Xs[rr], sum);
                    }
                } else {
                    for (int rb = wid; rb < RBN; rb += 8) {
                        T sum = pb[(rb * 8) * 32 + lane];
#pragma unroll
                        for (int w2 = 1; w2 < 8; ++w2) sum = Sc<T>::add(sum, pb[(rb * 8 + w2) * 32 + lane]);
                        const int rr = rb * 32 + lane;
                        const long row = row0 + rr;
                        if (row < n) {
                            const T q = Sc<T>::sub(Xs[rr], sum);
                            const T rv = reinterpret_cast<const T*>(xb + 1 * stride_x)[rr];
                            const T pv = reinterpret_cast<const T*>(xb + 2 * stride_x)[rr];
                            const T sv = reinterpret_cast<const T*>(xb + 3 * stride_x)[rr];
                            const T yv = reinterpret_cast<const T*>(xb + 4 * stride_x)[rr];
                            const T pn = Sc<T>::fma(beta, pv, rv);
                            const T sn = Sc<T>::fma(beta, sv, q);
                            p[row] = pn;
                            s[row] = sn;
                            y[row] = Sc<T>::fma(alpha, pn, yv);
                            r[row] = Sc<T>::sub(rv, Sc<T>::mul(alpha, sn));
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
        }
        if (MODE <= 1) {
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
                for (int q = 0; q < W; ++q) {
                    const double v = warp_sum(a[q]);
                    if (lane == 0 && jj < ncol) vals[(j0 + jj) * W + q] = v;
                }
            }
        }
    }
    if (MODE == 3) return;
    if (MODE == 2) {
        if (blockIdx.x == 0 && tid == 0) {
            st->gamma_prev = st->gamma;
            st->alpha_prev = st->alpha;
            st->it = st->it + 1;
        }
        return;
    }
    __syncthreads();
    if (!grid_commit(red, vals, C * W)) return;
    grid_finish(red, C * W, out);
}

}  // namespace rd
