// One-launch recycled CG / COCG iteration: the update of iteration i fused with
// the stencil, merged dots and first projection of iteration i+1, so the
// recycle basis K crosses HBM ONCE per iteration instead of twice.
//
// The unfused iteration (recycled_cg in romdot.cu; the CPU checker restates
// the same recurrence) is
//   cg_stencil_dots : w = A r ; {r^T r, r^T w, r^H r} ; alpha, beta
//   ts_tma<0>       : c1 = K^T w                       (K stream 1)
//   ts_tma<2>       : q = w - K (2 c1 - G c1) ; p, s, y, r updates (K stream 2)
// Row tile t of K is needed by the update (phase 1) and, for the next
// iteration, by c1' = K_t^T (A r')_t (phase 2). A r' at the rows of tile t
// needs r' at the stencil neighbours, at most P = N0*N1 rows (3D; N0 in 2D)
// away, so phase 2 of tile t can run as soon as phase 1 of every tile up to
// row t*TR + TR - 1 + P has run -- about ONE PLANE later. Every CTA marches its
// round-robin tiles (tile t -> CTA t % G, step t / G) through phase 1 and
// trails phase 2 by L = ceil((P + TR) / (TR G)) steps, so the second read of
// tile t comes from L2 (one plane of K: 18 MB at 128^3, c = 69, complex) rather
// than HBM. Cross-CTA order is a per-step counter that the owner warps bump
// (release) after writing r' and that the stencil warps poll (acquire) before
// reading r' halos through L2 (ld.global.cg).
//
// Warp roles (480 threads, one persistent CTA per SM):
//   warps 0-7  consumers: phase 1 (N-pass partial row sums of ts_tma MODE 2) and
//              phase 2 (T pass c1 += K_t^T w'_t, = MODE 0) from the TMA ring
//   warp  8    producer: one lane issues the TMA bulk copies for both phases
//   warps 9-12 stencil: w'_t = A r' for phase-2 tiles (round-robin), the
//              merged dots {r'^T r', r'^T w', r'^H r'}, w' to HBM and to a
//              shared-memory slot for the consumers
//   warp  13   release: gpu-scope fence + step counters after phase 1 of steps
//   warp  14   update: phase-1 reduction of the consumers' partials + CG update
// The last CTA reduces {c1 (C W), dots (2W+1)} in fixed order and runs the
// Chronopoulos-Gear scalar step (cg_recurrence) for the next launch.
#pragma once

#include "ts_tma.cuh"

namespace rd {

constexpr int FU_CONS = 256;                      // 8 consumer warps
constexpr int FU_NSW = 4;                         // stencil warps
constexpr int FU_NREL = 2;  // release warps (alternating steps: their fences overlap)
constexpr int FU_THREADS = FU_CONS + 32 + 32 * FU_NSW + 32 * FU_NREL + 32;  // + producer, stencil, release, update
constexpr int FU_REL_WARP = FU_CONS / 32 + 1 + FU_NSW;
constexpr int FU_UPD_WARP = FU_REL_WARP + FU_NREL;
constexpr int FU_NUPD = 1;
constexpr int FU_NPB = 2;  // phase-1 partial buffers
constexpr int FU_NWS = 2 * FU_NSW;                // w' slots (2 per stencil warp)

struct FusedLayout {
    int TR, S, RBN, L, LI, PF;  // PF: phase-1 L2 prefetch distance (steps)
    int poll_ns;                // back-off of the stencil warps' step-counter polls
    int rel_ns;                 // back-off of the release warps' wait for the update warp
    int ahead;                  // stencil polls look past the step they need
    int relbatch;               // release warps publish all their completed steps per fence
    // LI: item-order lead of phase 1 (>= L, slack for the stencil warps)
    int dbg;  // timing experiments only: bit 0 skips the step waits, bit 1 the stencil loads, bit 2 the phase-2 K reload
    uint32_t tile_bytes, x_bytes, stage_bytes;
    uint32_t off_ring, off_part, off_cw, off_vals, off_ws, off_dsc, off_bar, total;
};

template <class T> inline FusedLayout fused_layout(int C, int TR, int S) {
    FusedLayout L{};
    const uint32_t es = sizeof(T);
    auto al = [](uint32_t v) { return (v + 127u) & ~127u; };
    L.TR = TR;
    L.S = S;
    L.RBN = TR / 32;
    L.tile_bytes = (uint32_t)TR * C * es;
    L.x_bytes = (uint32_t)TR * es;
    L.stage_bytes = al(L.tile_bytes) + 5 * al(L.x_bytes);
    uint32_t o = 0;
    L.off_ring = o;
    o += L.stage_bytes * S;
    L.off_part = o;
    o += al((uint32_t)FU_NPB * TR * 9 * es);  // phase-1 partials [row][9]
    L.off_cw = o;
    o += al((uint32_t)2 * C * es);  // coef, staged c1
    L.off_vals = o;
    o += al((uint32_t)(C * Sc<T>::W + 2 * Sc<T>::W + 1) * sizeof(double));
    L.off_ws = o;
    o += al(L.x_bytes) * FU_NWS;
    L.off_dsc = o;
    o += al(FU_NSW * 8 * sizeof(double));
    L.off_bar = o;
    o += (2 * S + 2 * FU_NWS + 2 * FU_NPB) * 8;
    L.total = o;
    return L;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_gpu(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_cta_shared(unsigned* p, unsigned v) {
    asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Optional per-role cycle accounting (ROMDOT_FUSED_PROF=1): lane 0 of each
// warp adds its wait / total cycles to tprof[slot] (summed over CTAs, warps).
struct FuProf {
    unsigned long long* t;
    unsigned long long acc[8];
    long long t0;
    __device__ void start() {
        for (int i = 0; i < 8; ++i) acc[i] = 0;
        t0 = clock64();
    }
    __device__ long long now() const { return t ? clock64() : 0; }
    __device__ void add(int i, long long a) {
        if (t) acc[i] += (unsigned long long)(clock64() - a);
    }
    __device__ void flush(int base, bool lead) {
        if (!t || !lead) return;
        acc[7] = (unsigned long long)(clock64() - t0);
        for (int i = 0; i < 8; ++i) atomicAdd(t + base + i, acc[i]);
    }
};

template <class T> __device__ __forceinline__ T ldcg_(const T* p);
template <> __device__ __forceinline__ double ldcg_<double>(const double* p) { return __ldcg(p); }
template <> __device__ __forceinline__ cplx ldcg_<cplx>(const cplx* p) { return __ldcg(p); }

// Row p of A x with x read through L2 (written by other CTAs in this launch);
// same loads and summation order as zmarch (kernels.cuh). Split in two so the
// coefficient loads (constant fields, HBM) can be issued before the stencil
// warp waits for the step counters, and only the x loads follow the wait.
struct StCoef {
    double dg, fxm, fxp, fym, fyp, fzm, fzp;
    long s1, s2;
    unsigned char m;  // neighbour mask: x-, x+, y-, y+, z-, z+
};

__device__ __forceinline__ StCoef stencil_coef(const OpDev& op, long p) {
    StCoef c;
    const long n = op.n;
    c.s1 = op.N0;
    c.s2 = (long)op.N0 * op.N1;
    const double* __restrict__ Fd = op.F;
    const long q = p / op.N0;
    const int i = (int)(p - q * op.N0);
    const int j = (int)(q % op.N1);
    const int k = (int)(q / op.N1);
    const bool three = op.d == 3;
    const bool hx_m = i > 0, hx_p = i < op.N0 - 1, hy_m = j > 0, hy_p = j < op.N1 - 1;
    const bool hz_m = three && k > 0, hz_p = three && k < op.N2 - 1;
    c.m = (unsigned char)(hx_m | hx_p << 1 | hy_m << 2 | hy_p << 3 | hz_m << 4 | hz_p << 5);
    c.fzm = hz_m ? __ldg(Fd + 3 * n + p - c.s2) : 0.0;
    c.fzp = hz_p ? __ldg(Fd + 3 * n + p) : 0.0;
    c.dg = __ldg(Fd + p);
    c.fxm = hx_m ? __ldg(Fd + n + p - 1) : 0.0;
    c.fxp = hx_p ? __ldg(Fd + n + p) : 0.0;
    c.fym = hy_m ? __ldg(Fd + 2 * n + p - c.s1) : 0.0;
    c.fyp = hy_p ? __ldg(Fd + 2 * n + p) : 0.0;
    return c;
}

template <class T>
__device__ __forceinline__ T stencil_apply_l2(const OpDev& op, const T* x, long p, const StCoef& c, T& xc) {
    const bool three = op.d == 3;
    const T xm = (c.m & 16) ? ldcg_(x + p - c.s2) : Sc<T>::zero();
    xc = ldcg_(x + p);
    const T xp = (c.m & 32) ? ldcg_(x + p + c.s2) : Sc<T>::zero();
    const T xim = (c.m & 1) ? ldcg_(x + p - 1) : Sc<T>::zero();
    const T xip = (c.m & 2) ? ldcg_(x + p + 1) : Sc<T>::zero();
    const T xjm = (c.m & 4) ? ldcg_(x + p - c.s1) : Sc<T>::zero();
    const T xjp = (c.m & 8) ? ldcg_(x + p + c.s1) : Sc<T>::zero();
    T acc = Sc<T>::zero();
    acc = axpy_real(c.fxm, xim, acc);
    acc = axpy_real(c.fxp, xip, acc);
    acc = axpy_real(c.fym, xjm, acc);
    acc = axpy_real(c.fyp, xjp, acc);
    if (three) {
        acc = axpy_real(c.fzm, xm, acc);
        acc = axpy_real(c.fzp, xp, acc);
    }
    return Sc<T>::sub(diag_apply<T>(c.dg, op.shift, xc), acc);
}

// Item order shared by the producer and the consumers: phase 1 of steps
// 0..L first, then phase 2 of step s followed by phase 1 of step s + L + 1.
// Phase 2 of step s waits (through the step counters) for phase 1 of steps up
// to s + L on every CTA, all of which precede it in every CTA's order, so the
// march cannot deadlock (all CTAs are co-resident: grid <= SMs, 1 CTA / SM).
template <class F> __device__ __forceinline__ void fused_items(int ns, int L, F&& f) {
    int s1 = 0;
    for (; s1 <= L && s1 < ns; ++s1) f(1, s1);  // L = the layout's LI
    for (int s2 = 0; s2 < ns; ++s2) {
        f(2, s2);
        if (s1 < ns) {
            f(1, s1);
            ++s1;
        }
    }
}

template <class T, int CPW>
__global__ void __launch_bounds__(FU_THREADS, 1)
    cg_fused(OpDev op, const T* __restrict__ Krb, int C, long ntile, FusedLayout FL, T* w, T* r, T* p, T* s, T* y,
             CGState* st, double* hist, GridRed red, double* cbuf, unsigned* stepcnt, const T* __restrict__ G,
             unsigned long long* tprof, unsigned* chk, unsigned epoch) {
    // Programmatic dependent launch (ROMDOT_FUSED_PDL=1, opt-in): the next
    // iteration's launch may be scheduled as soon as every CTA of this one has
    // started, so its CTAs take the SMs this grid's CTAs free while the last CTA
    // reduces, and wait here until this grid has completed (memory visible).
    // Nothing before the wait reads global memory. Without the launch
    // attribute both instructions are no-ops.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (st->done) return;
    // ROMDOT_FUSED_PROF: launch-phase timestamps (ns) min/max over CTAs in
    // tprof[40..47], folded into per-launch sums in tprof[48..55] by the last CTA
    auto gtime = [] {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
    if (tprof && threadIdx.x == 0) {
        const unsigned long long t = gtime();
        atomicMin(tprof + 40, t);
        atomicMax(tprof + 41, t);
    }
    constexpr int W = Sc<T>::W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int TR = FL.TR, S = FL.S, RBN = FL.RBN;
    const long n = op.n;
    const int Gd = gridDim.x, bid = blockIdx.x;
    const int ns = (int)((ntile - bid + Gd - 1) / Gd);  // steps in which this CTA owns a tile
    const long nsteps = (ntile + Gd - 1) / Gd;
    const uint32_t xs_stride = (FL.x_bytes + 127u) & ~127u;
    const uint32_t k_stride = (FL.tile_bytes + 127u) & ~127u;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + FL.off_bar);
    uint64_t* empty = full + S;
    uint64_t* wfull = empty + S;
    uint64_t* wempty = wfull + FU_NWS;
    uint64_t* pready = wempty + FU_NWS;  // partials of a phase-1 item written (consumers)
    uint64_t* pfree = pready + FU_NPB;   // ... and consumed (update warp)
    T* part = reinterpret_cast<T*>(smem + FL.off_part);
    T* cw = reinterpret_cast<T*>(smem + FL.off_cw);
    T* c1s = cw + C;
    double* vals = reinterpret_cast<double*>(smem + FL.off_vals);
    double* dsc = reinterpret_cast<double*>(smem + FL.off_dsc);
    __shared__ unsigned relcnt[1];  // phase-1 items stored by the update warp
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long P = op.d == 3 ? (long)op.N0 * op.N1 : (long)op.N0;
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], FU_CONS / 32 + FU_NUPD);  // consumers + update warps
        }
        for (int i = 0; i < FU_NWS; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], FU_CONS / 32);
        }
        for (int i = 0; i < FU_NPB; ++i) {
            mbar_init(&pready[i], FU_CONS / 32);
            mbar_init(&pfree[i], 1);
        }
        fence_mbar_init();
        relcnt[0] = 0u;
    }
    for (int t = tid; t < C; t += blockDim.x) c1s[t] = Sc<T>::get(cbuf + (size_t)t * W);
    __syncthreads();  // barriers initialised, c1 staged
    if (wid != FU_CONS / 32) {
        // coef = 2 c1 - G c1 (the one-pass projection's Gram-corrected
        // coefficient; G = K^T K symmetric), c1 = K^T w of the previous launch /
        // the prologue. One warp per row of G (coalesced, fixed order); the
        // producer warp is already issuing its first TMA loads meanwhile.
        constexpr int NW = FU_THREADS / 32 - 1;
        const int q = wid < FU_CONS / 32 ? wid : wid - 1;
        // three rows per pass with all their loads in flight (C <= 128: <= 4 per lane and row)
        for (int t0 = q; t0 < C; t0 += 3 * NW) {
            T acc[3] = {Sc<T>::zero(), Sc<T>::zero(), Sc<T>::zero()};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = lane + 32 * u;
                if (j < C) {
                    const T cj = c1s[j];
#pragma unroll
                    for (int v = 0; v < 3; ++v) {
                        const int t = t0 + v * NW;
                        if (t < C) acc[v] = Sc<T>::fma(__ldg(G + (size_t)t * C + j), cj, acc[v]);
                    }
                }
            }
#pragma unroll
            for (int v = 0; v < 3; ++v) {
                const int t = t0 + v * NW;
                if constexpr (W == 1) {
                    acc[v] = warp_sum(acc[v]);
                } else {
                    ((cplx&)acc[v]).x = warp_sum(((cplx&)acc[v]).x);
                    ((cplx&)acc[v]).y = warp_sum(((cplx&)acc[v]).y);
                }
                if (lane == 0 && t < C) cw[t] = Sc<T>::sub(Sc<T>::scale(c1s[t], 2.0), acc[v]);
            }
        }
        // named barrier 1 over every warp but the producer
        asm volatile("bar.sync 1, %0;" ::"r"(FU_THREADS - 32) : "memory");
    }
    if (tprof && tid == 0) atomicMax(tprof + 42, gtime());

    if (wid == FU_CONS / 32) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            FuProf pr{tprof};
            pr.start();
            int k = 0;
            uint32_t kph = 0;  // ring slot and its phase parity
            uint64_t pol_last, pol_first;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
            fused_items(ns, FL.LI, [&](int ph, int sidx) {
                const long t = (long)sidx * Gd + bid;
                const int stage = k;
                const uint32_t use = kph;
                if (++k == S) {
                    k = 0;
                    kph ^= 1u;
                }
                long long ta = pr.now();
                mbar_wait(&empty[stage], (use & 1u) ^ 1u);
                pr.add(0, ta);
                unsigned char* sb = smem + FL.off_ring + (size_t)stage * FL.stage_bytes;
                if (ph == 1) {
                    // L2 prefetch of the phase-1 tile PF steps ahead: keeps HBM
                    // requests in flight beyond what the shared-memory ring holds
                    // (half of the ring carries the L2-resident phase-2 tiles)
                    if (FL.PF > 0 && sidx + FL.PF < ns) {
                        const long tp = (long)(sidx + FL.PF) * Gd + bid;
                        prefetch_l2(Krb + (size_t)tp * TR * C, FL.tile_bytes);
                        prefetch_l2(w + (size_t)tp * TR, FL.x_bytes);
                        prefetch_l2(r + (size_t)tp * TR, FL.x_bytes);
                        prefetch_l2(p + (size_t)tp * TR, FL.x_bytes);
                        prefetch_l2(s + (size_t)tp * TR, FL.x_bytes);
                        prefetch_l2(y + (size_t)tp * TR, FL.x_bytes);
                    }
                    mbar_arrive_expect_tx(&full[stage], FL.tile_bytes + 5 * FL.x_bytes);
                    // phase 1 reads the tile from HBM and keeps it in L2 (evict_last)
                    // for its phase-2 re-read about L steps later
                    if (FL.dbg & 32)
                        tma_load_1d(sb, Krb + (size_t)t * TR * C, FL.tile_bytes, &full[stage]);
                    else
                        tma_load_1d_hint(sb, Krb + (size_t)t * TR * C, FL.tile_bytes, &full[stage], pol_last);
                    unsigned char* xb = sb + k_stride;
                    tma_load_1d(xb, w + (size_t)t * TR, FL.x_bytes, &full[stage]);
                    tma_load_1d(xb + 1 * xs_stride, r + (size_t)t * TR, FL.x_bytes, &full[stage]);
                    tma_load_1d(xb + 2 * xs_stride, p + (size_t)t * TR, FL.x_bytes, &full[stage]);
                    tma_load_1d(xb + 3 * xs_stride, s + (size_t)t * TR, FL.x_bytes, &full[stage]);
                    tma_load_1d(xb + 4 * xs_stride, y + (size_t)t * TR, FL.x_bytes, &full[stage]);
                } else if (FL.dbg & 4) {
                    mbar_arrive(&full[stage]);
                } else {
                    mbar_arrive_expect_tx(&full[stage], FL.tile_bytes);
                    if (FL.dbg & 32)
                        tma_load_1d(sb, Krb + (size_t)t * TR * C, FL.tile_bytes, &full[stage]);
                    else
                        tma_load_1d_hint(sb, Krb + (size_t)t * TR * C, FL.tile_bytes, &full[stage], pol_first);
                }
            });
            pr.flush(0, true);
        }
    } else if (wid >= FU_REL_WARP && wid < FU_REL_WARP + FU_NREL) {
        // ------------------------------ release warp ------------------------------
        // Publishes phase 1 of each step to the other CTAs: waits until the
        // update warp has stored r', p, s, y of the step's tile (CTA-scope
        // counter), then ONE gpu-scope fence (cumulative over those stores) for
        // every step completed since the last one, and the step counters. (A
        // fence per step in the update warp itself measured slower: 0.9 us each.)
        // FU_NREL warps take alternating steps so consecutive fences overlap (a
        // fence also waits for the warp's previous step-counter add).
        // FL.relbatch: one fence publishes EVERY step of this warp's parity that
        // the update warp has completed by then (the fence, ~1.6 us under load,
        // is the publication chain's throughput limit when steps arrive faster).
        if (lane == 0) {
            FuProf pr{tprof};
            pr.start();
            volatile unsigned* rc = relcnt;
            for (int s1 = wid - FU_REL_WARP; s1 < ns;) {
                long long ta = pr.now();
                unsigned done;
                while ((done = *rc) < (unsigned)(s1 + 1)) __nanosleep(FL.rel_ns);
                pr.add(0, ta);
                ta = pr.now();
                fence_acq_rel_gpu();
                const int hi = FL.relbatch ? min((int)done, ns) : s1 + 1;
                for (; s1 < hi; s1 += FU_NREL) red_relaxed_gpu(stepcnt + s1, 1u);
                pr.add(1, ta);
                if (pr.t) pr.acc[2] += 1900;  // fence count (x 1 us in the report)
            }
            pr.flush(8, wid == FU_REL_WARP);
        }
    } else if (wid == FU_UPD_WARP) {
        // ------------------------------ update warp ------------------------------
        // Phase 1 after the consumers' partial row sums: q = w - sum of the 8
        // column-block partials (fixed order), then the CG update of p, s, y, r
        // for the tile's rows (lane = row). Runs beside the consumers, which
        // never wait for it (FU_NPB partial buffers).
        FuProf pr{tprof};
        pr.start();
        const T alpha = ld2<T>(st->alpha), beta = ld2<T>(st->beta);
        int k = 0, k1 = 0;
        uint32_t kph = 0;
        fused_items(ns, FL.LI, [&](int ph, int sidx) {
            const int stage = k;
            const uint32_t use = kph;
            if (++k == S) {
                k = 0;
                kph ^= 1u;
            }
            long long ta = pr.now();
            mbar_wait(&full[stage], use & 1u);  // the stage holds this item (empty phase alignment)
            pr.add(0, ta);
            if (ph == 1) {
                const unsigned char* xb = smem + FL.off_ring + (size_t)stage * FL.stage_bytes + k_stride;
                const int pbi = k1 % FU_NPB;
                const T* pb = part + (size_t)pbi * TR * 9;
                ta = pr.now();
                mbar_wait(&pready[pbi], (uint32_t)(k1 / FU_NPB) & 1u);
                pr.add(1, ta);
                ta = pr.now();
                const long row0 = (long)sidx * Gd * TR + (long)bid * TR;
                for (int rr = lane; rr < TR; rr += 32) {
                    const T* pr9 = pb + rr * 9;
                    const T sum = Sc<T>::add(Sc<T>::add(Sc<T>::add(pr9[0], pr9[1]), Sc<T>::add(pr9[2], pr9[3])),
                                             Sc<T>::add(Sc<T>::add(pr9[4], pr9[5]), Sc<T>::add(pr9[6], pr9[7])));
                    const long row = row0 + rr;
                    if (row < n && !(FL.dbg & 16)) {
                        const T q = Sc<T>::sub(reinterpret_cast<const T*>(xb)[rr], sum);
                        const T rv = reinterpret_cast<const T*>(xb + 1 * xs_stride)[rr];
                        const T pv = reinterpret_cast<const T*>(xb + 2 * xs_stride)[rr];
                        const T sv = reinterpret_cast<const T*>(xb + 3 * xs_stride)[rr];
                        const T yv = reinterpret_cast<const T*>(xb + 4 * xs_stride)[rr];
                        const T pn = Sc<T>::fma(beta, pv, rv);
                        const T sn = Sc<T>::fma(beta, sv, q);
                        p[row] = pn;
                        s[row] = sn;
                        y[row] = Sc<T>::fma(alpha, pn, yv);
                        r[row] = Sc<T>::sub(rv, Sc<T>::mul(alpha, sn));
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    // ROMDOT_FUSED_CHECK: tile epoch, published by the same release
                    // chain as the r' rows it vouches for
                    if (chk) chk[16 + (long)sidx * Gd + bid] = epoch;
                    mbar_arrive(&pfree[pbi]);
                    red_release_cta_shared(relcnt, 1u);
                }
                pr.add(2, ta);
                ++k1;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
        });
        pr.flush(16, lane == 0);
    } else if (wid > FU_CONS / 32) {
        // ------------------------------ stencil warps ------------------------------
        const int sw = wid - FU_CONS / 32 - 1;  // phase-2 steps s2 = sw mod FU_NSW
        T g = Sc<T>::zero(), dl = Sc<T>::zero();
        double h = 0.0;
        long ok = -1;  // step counters verified complete through this step
        int k = 0;
        FuProf pr{tprof};
        pr.start();
        for (int s2 = sw; s2 < ns; s2 += FU_NSW, ++k) {
            const long t = (long)s2 * Gd + bid;
            long thi = (t * TR + TR - 1 + P) / TR;
            if (thi > ntile - 1) thi = ntile - 1;
            const long shi = thi / Gd;
            // coefficients of the first row block before the wait (no dependence)
            const long row_first = t * TR + lane;
            StCoef cf = stencil_coef(op, row_first < n ? row_first : n - 1);
            long long ta = pr.now();
            // the step counters from ok+1 on, one per lane, polled in parallel (one
            // L2 round trip per check instead of one per step); acquire loads so
            // the r' halo loads below are ordered after the releases they observe.
            // With ROMDOT_FUSED_AHEAD (default) a poll also looks past shi and
            // advances ok over every consecutive complete step, so later tiles of
            // this warp usually find their steps covered without another poll.
            while (ok < shi && !(FL.dbg & 1)) {
                const long lim = FL.ahead ? nsteps - 1 : shi;
                const int nq = (int)(lim - ok < 32 ? lim - ok : 32);
                bool good = true;
                if (lane < nq) {
                    const long sq = ok + 1 + lane;
                    const long tiles = ntile - sq * Gd < Gd ? ntile - sq * Gd : Gd;
                    good = ld_acquire_u32(stepcnt + sq) >= (unsigned)tiles;  // one release per CTA and step
                }
                const unsigned bad = __ballot_sync(0xffffffffu, !good);
                ok += bad ? __ffs(bad) - 1 : nq;
                if (ok < shi) __nanosleep(FL.poll_ns);
            }
            pr.add(0, ta);
            if (chk) {
                // protocol check: every tile this warp's rows read r' from (the row
                // itself and its six stencil neighbours) must carry this launch's
                // epoch once the step counters say so; a stale epoch is a halo read
                // that raced the owner's update (counted in chk[0])
                for (int rb = 0; rb < RBN; ++rb) {
                    const long row = t * TR + rb * 32 + lane;
                    if (row >= n) continue;
                    const StCoef cq = stencil_coef(op, row);
                    const long nb[7] = {row, row - 1, row + 1, row - cq.s1, row + cq.s1, row - cq.s2, row + cq.s2};
                    const bool use[7] = {true, (cq.m & 1) != 0, (cq.m & 2) != 0, (cq.m & 4) != 0,
                                         (cq.m & 8) != 0, (cq.m & 16) != 0, (cq.m & 32) != 0};
#pragma unroll
                    for (int q = 0; q < 7; ++q)
                        if (use[q] && ld_relaxed_u32(chk + 16 + nb[q] / TR) != epoch) atomicAdd(chk, 1u);
                }
            }
            const int slot = FU_NSW * (k & 1) + sw;
            const uint32_t use = (uint32_t)(k >> 1);
            ta = pr.now();
            mbar_wait(&wempty[slot], (use & 1u) ^ 1u);
            pr.add(1, ta);
            T* ws = reinterpret_cast<T*>(smem + FL.off_ws + (size_t)slot * xs_stride);
            ta = pr.now();
            for (int rb = 0; rb < RBN; ++rb) {
                const long row = t * TR + rb * 32 + lane;
                T wv = Sc<T>::zero();
                if (rb > 0) cf = stencil_coef(op, row < n ? row : n - 1);
                if (row < n) {
                    T rc;
                    if (FL.dbg & 2) {
                        rc = ldcg_(r + row);
                        wv = rc;
                    } else
                        wv = stencil_apply_l2<T>(op, r, row, cf, rc);
                    w[row] = wv;
                    g = Sc<T>::fma(rc, rc, g);
                    dl = Sc<T>::fma(rc, wv, dl);
                    h += Sc<T>::abs2(rc);
                }
                ws[rb * 32 + lane] = wv;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&wfull[slot]);
            pr.add(2, ta);
        }
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
        for (int q = 0; q < 2 * W + 1; ++q) {
            const double sum = warp_sum(v[q]);
            if (lane == 0) dsc[sw * 8 + q] = sum;
        }
        pr.flush(32, lane == 0);
    } else {
        // ------------------------------ consumers ------------------------------
        const int j0 = wid * CPW;
        int ncol = C - j0;
        if (ncol > CPW) ncol = CPW;
        T acc[CPW];
#pragma unroll
        for (int jj = 0; jj < CPW; ++jj) acc[jj] = Sc<T>::zero();
        int k = 0, k1 = 0, k2 = 0;
        uint32_t kph = 0;
        FuProf pr{tprof};
        pr.start();
        fused_items(ns, FL.LI, [&](int ph, int sidx) {
            const long t = (long)sidx * Gd + bid;
            const int stage = k;
            const uint32_t use = kph;
            if (++k == S) {
                k = 0;
                kph ^= 1u;
            }
            long long ta = pr.now();
            mbar_wait(&full[stage], use & 1u);
            pr.add(ph == 1 ? 0 : 1, ta);
            const unsigned char* sb = smem + FL.off_ring + (size_t)stage * FL.stage_bytes;
            const T* Ks = reinterpret_cast<const T*>(sb);
            if (ph == 2) {
                // T pass: c1 += K_t^T w'_t (w' from the stencil warp's slot)
                const int sw = k2 % FU_NSW, kk = k2 / FU_NSW;
                const int slot = FU_NSW * (kk & 1) + sw;
                ta = pr.now();
                mbar_wait(&wfull[slot], (uint32_t)(kk >> 1) & 1u);
                pr.add(2, ta);
                const T* Xs = reinterpret_cast<const T*>(smem + FL.off_ws + (size_t)slot * xs_stride);
                ta = pr.now();
                for (int rb = 0; rb < RBN; ++rb) {
                    const T xv = Xs[rb * 32 + lane];
                    const T* kb = Ks + (size_t)rb * 32 * C + lane;
#pragma unroll
                    for (int jj = 0; jj < CPW; ++jj)
                        if (jj < ncol) acc[jj] = opfma<T, false>(kb[(size_t)(j0 + jj) * 32], xv, acc[jj]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&wempty[slot]);
                pr.add(4, ta);
                ++k2;
            } else {
                // N pass (partial row sums of this warp's columns) of ts_tma MODE 2;
                // the update warp reduces them and applies the CG update.
                // Partials go to a [row][9] buffer (stride 9: conflict-free both ways).
                const int pbi = k1 % FU_NPB;
                T* pb = part + (size_t)pbi * TR * 9;
                ta = pr.now();
                mbar_wait(&pfree[pbi], ((uint32_t)(k1 / FU_NPB) & 1u) ^ 1u);
                pr.add(3, ta);
                long long tb = pr.now();
                for (int rb = 0; rb < RBN; ++rb) {
                    const T* kb = Ks + (size_t)rb * 32 * C + lane;
                    // two independent chains (latency: one chain of 2*CPW dependent DFMAs)
                    T pa0 = Sc<T>::zero(), pa1 = Sc<T>::zero();
#pragma unroll
                    for (int jj = 0; jj < CPW; jj += 2) {
                        if (jj < ncol) pa0 = Sc<T>::fma(kb[(size_t)(j0 + jj) * 32], cw[j0 + jj], pa0);
                        if (jj + 1 < CPW && jj + 1 < ncol)
                            pa1 = Sc<T>::fma(kb[(size_t)(j0 + jj + 1) * 32], cw[j0 + jj + 1], pa1);
                    }
                    pb[(rb * 32 + lane) * 9 + wid] = Sc<T>::add(pa0, pa1);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&pready[pbi]);
                pr.add(5, tb);
                ++k1;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
        });
        pr.flush(24, lane == 0);
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
    __syncthreads();
    if (tprof && tid == 0) {
        const unsigned long long t = gtime();
        atomicMin(tprof + 43, t);
        atomicMax(tprof + 44, t);
    }
    const int nv = C * W + 2 * W + 1;
    if (tid < 2 * W + 1) {
        double a = dsc[tid];
#pragma unroll
        for (int q = 1; q < FU_NSW; ++q) a += dsc[q * 8 + tid];
        vals[C * W + tid] = a;
    }
    __syncthreads();
    if (!grid_commit(red, vals, nv)) return;
    grid_finish(red, nv, cbuf);
    // every CTA has committed: reset the step counters for the next launch
    for (long q = tid; q < nsteps; q += blockDim.x) stepcnt[q] = 0u;
    if (tid == 0) {
        __threadfence();
        st->gamma_prev = st->gamma;
        st->alpha_prev = st->alpha;
        st->it = st->it + 1;
        cg_recurrence<T>(st, cbuf + C * W, hist);
        if (tprof) {
            // per launch: entry spread, prologue, roles (first/last CTA), commit+finish
            const unsigned long long t = gtime(), a = tprof[40], b = tprof[41], c = tprof[42], d = tprof[43],
                                     e = tprof[44];
            tprof[48] += b - a;
            tprof[49] += c - a;
            tprof[50] += d - c;
            tprof[51] += e - c;
            tprof[52] += t - e;
            tprof[53] += t - a;
            if (tprof[45] && a - tprof[45] < 1000000ull) {  // previous launch end -> this entry (same solve)
                tprof[54] += a - tprof[45];
                tprof[55] += 1;
            }
            tprof[46] += 1;  // launches that ran (not the no-ops after convergence)
            tprof[45] = t;
            tprof[40] = ~0ull;
            tprof[41] = 0;
            tprof[42] = 0;
            tprof[43] = ~0ull;
            tprof[44] = 0;
        }
    }
}

}  // namespace rd
