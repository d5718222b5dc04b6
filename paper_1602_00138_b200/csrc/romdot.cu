// Host runtime of the B200 basis builder: context, device operator, recycled
// CG / COCG driver, device GlobalBasis, process_system and the C ABI
// (include/romdot_b200.h). All control flow that the reference runs in
// src/basis.cpp and src/krylov.cpp lives here in C++; all arithmetic on
// n-vectors runs in the kernels of kernels.cuh / dense.cuh.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/romdot_b200.h"
#include "dense.cuh"
#include "kernels.cuh"
#include "ts_tma.cuh"
#include "cg_fused.cuh"
#include "bcg_defl.cuh"
#include "stencil_tma.cuh"
#include "rom.cuh"

namespace rd {

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct SolverError : std::runtime_error {
    explicit SolverError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {  // types.hpp:28-30, exit code 4
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};

static thread_local std::string g_err;

// ROMDOT_VERBOSE=1 prints solver progress to stderr (host-side, no device syncs added).
static int verbose() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("ROMDOT_VERBOSE");
        v = e ? std::atoi(e) : 0;
    }
    return v;
}
#define VLOG(lvl, ...)                           \
    do {                                         \
        if (verbose() >= (lvl)) {                \
            std::fprintf(stderr, "[romdot] ");   \
            std::fprintf(stderr, __VA_ARGS__);   \
            std::fprintf(stderr, "\n");          \
            std::fflush(stderr);                 \
        }                                        \
    } while (0)

#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + ":" + \
                            std::to_string(__LINE__));                                               \
    } while (0)

// ROMDOT_VERBOSE>=3: bitwise-sensitive checksum of a device buffer (debug of
// determinism; copies to host, slow).
// Level 4: non-perturbing trace. Each checkpoint enqueues an order-independent
// exact hash (sum of position-mixed 64-bit words) into a device log on the
// stream -- no host syncs -- and dbg_flush prints the log at a point where the
// caller syncs anyway (end of process_system).
__global__ void dbg_hash_kernel(const unsigned long long* w, long nw, unsigned long long* slot) {
    unsigned long long acc = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nw; i += (long)gridDim.x * blockDim.x) {
        unsigned long long z = w[i] ^ ((unsigned long long)i * 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        acc += z ^ (z >> 31);
    }
    atomicAdd(slot, acc);
}
struct DbgLog {
    unsigned long long* d = nullptr;
    std::vector<std::string> names;
    static constexpr int kCap = 1 << 16;
};
static DbgLog& dbg_log() {
    static DbgLog L;
    return L;
}
static void dbg_flush(cudaStream_t s) {
    DbgLog& L = dbg_log();
    if (verbose() < 4 || !L.d || L.names.empty()) return;
    std::vector<unsigned long long> h(L.names.size());
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), L.d, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < h.size(); ++i) std::fprintf(stderr, "[romdot-hash] %s %016llx\n", L.names[i].c_str(), h[i]);
    cudaMemsetAsync(L.d, 0, sizeof(unsigned long long) * h.size(), s);
    L.names.clear();
}

template <class T> static void dbg_sum(const char* tag, const T* p, long count, cudaStream_t s) {
    if (verbose() < 3 || !p || count <= 0) return;
    if (verbose() >= 4) {
        DbgLog& L = dbg_log();
        if (!L.d) {
            cudaMalloc(&L.d, sizeof(unsigned long long) * DbgLog::kCap);
            cudaMemset(L.d, 0, sizeof(unsigned long long) * DbgLog::kCap);
        }
        if ((int)L.names.size() >= DbgLog::kCap) return;
        const long nw = (long)(sizeof(T) * count / 8);
        dbg_hash_kernel<<<64, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(p), nw, L.d + L.names.size());
        L.names.push_back(tag);
        return;
    }
    std::vector<T> h(count);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), p, sizeof(T) * count, cudaMemcpyDeviceToHost);
    unsigned long long x = 1469598103934665603ull;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(h.data());
    for (size_t i = 0; i < sizeof(T) * (size_t)count; ++i) x = (x ^ b[i]) * 1099511628211ull;
    long nonfinite = 0;  // with ROMDOT_POISON=1: reads of never-written device memory surface here
    const double* dv = reinterpret_cast<const double*>(h.data());
    std::string where;
    for (size_t i = 0; i < sizeof(T) * (size_t)count / sizeof(double); ++i)
        if (!std::isfinite(dv[i])) {
            if (nonfinite < 12) where += " " + std::to_string(i);
            ++nonfinite;
        }
    std::fprintf(stderr, "[romdot-sum] %s %016llx%s\n", tag, x,
                 nonfinite ? (" NONFINITE " + std::to_string(nonfinite) + " at doubles" + where).c_str() : "");
}

template <class T> constexpr int dt_of();
template <> constexpr int dt_of<double>() { return 0; }
template <> constexpr int dt_of<cplx>() { return 1; }

// ------------------------------------------------------------- buffers ---
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    // cudaFree does not wait for work queued on the library's non-blocking
    // stream: a buffer is only released after the device has drained, so a
    // kernel still in flight never reads freed (and possibly reused) memory.
    ~DevBuf() {
        if (p) {
            cudaDeviceSynchronize();
            cudaFree(p);
        }
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(p));
        }
        p = nullptr;
        CK(cudaMalloc(&p, b));
        bytes = b;
        // ROMDOT_POISON=1: fill fresh allocations with NaN bytes so any read of
        // unwritten device memory surfaces as a NaN in a normal-speed run (the
        // GPU pool refuses compute-sanitizer: profiles/r02_sanitizer_refused.txt).
        static const int poison = [] {
            const char* e = std::getenv("ROMDOT_POISON");
            return e ? std::atoi(e) : 0;
        }();
        if (poison) {
            // cudaMemset on device memory returns before the fill has run, and the fill sits on
            // the legacy default stream, which the library's non-blocking stream does not wait
            // for: without the sync the NaN fill can land AFTER the first writes to the buffer
            CK(cudaMemset(p, 0xFF, b));
            CK(cudaDeviceSynchronize());
        }
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// ------------------------------------------------------------- context ---
struct Ctx {
    int device = 0;
    int sms = 148;
    int solver = 0;  // 0: recycled CG / COCG (default), 1: the reference's recycled MINRES (real, parity path)
    cudaStream_t s = nullptr;
    DevBuf partials, counter, scal, cgst, hist, rflag;
    DevBuf fstep;  // per-step counters of the fused iteration (zero between launches)
    DevBuf fprof;  // ROMDOT_FUSED_PROF: per-role cycle sums of cg_fused
    DevBuf fchk;   // ROMDOT_FUSED_CHECK: [0] stale-halo count, [16 + tile] tile epochs
    unsigned fchk_epoch = 0;
    long fchk_violations = 0, fchk_checked = 0;  // totals over the context's solves
    long fprof_launches = 0;
    // print and reset the cg_fused role accounting (average per launch, per warp)
    void fprof_reset() {
        unsigned long long h[56] = {};
        h[40] = h[43] = ~0ull;
        CK(cudaMemcpy(fprof.p, h, sizeof(h), cudaMemcpyHostToDevice));
    }
    void fprof_report() {
        if (!fprof.p || !fprof_launches) return;
        unsigned long long h[56];  // 5 roles x 8 slots + launch-phase timestamps
        CK(cudaMemcpy(h, fprof.p, sizeof(h), cudaMemcpyDeviceToHost));
        const double L = h[46] ? (double)h[46] : (double)fprof_launches;  // launches that ran
        auto pr = [&](const char* role, int base, double warps, const char* const* names) {
            std::fprintf(stderr, "[cg_fused] %-9s", role);
            for (int i = 0; i < 8; ++i)
                if (names[i]) std::fprintf(stderr, " %s=%.1fus", names[i], h[base + i] / L / warps / 1.9e3);
            std::fprintf(stderr, "\n");
        };
        const double G = sms;
        static const char* const np[8] = {"wait_empty", nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, "total"};
        static const char* const nr[8] = {"wait_owners", "fence+atomic", "batches(us=count)", nullptr, nullptr, nullptr, nullptr, "total"};
        static const char* const ns[8] = {"poll", "wait_slot", "compute", nullptr, nullptr, nullptr, nullptr, "total"};
        static const char* const nc[8] = {"full_p1", "full_p2", "wfull", "pfree", "p2_math", "p1_partial", nullptr, "total"};
        static const char* const nu[8] = {"full", "pready", "update", "fence+red", nullptr, nullptr, nullptr, "total"};
        pr("producer", 0, G, np);
        pr("release", 8, G, nr);
        pr("update", 16, G, nu);
        pr("stencil", 32, G * 4, ns);
        pr("consumer", 24, G * 8, nc);
        std::fprintf(stderr,
                     "[cg_fused] launch    entry_spread=%.1fus prologue=%.1fus roles_first=%.1fus roles_last=%.1fus "
                     "commit+finish=%.1fus span=%.1fus gap_prev_end=%.1fus\n",
                     h[48] / L / 1e3, h[49] / L / 1e3, h[50] / L / 1e3, h[51] / L / 1e3, h[52] / L / 1e3,
                     h[53] / L / 1e3, h[55] ? (double)h[54] / h[55] / 1e3 : 0.0);
        fprof_reset();
        fprof_launches = 0;
    }
    CGState* st_host = nullptr;  // pinned, 2 slots
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t mark[2] = {nullptr, nullptr};
    int nmark = 0;
    long launches = 0;
    int hist_cap = 1 << 16;

    // Sampled per-kernel-class device timing (CUDA events on this stream):
    // the first inner iteration of every launch batch is bracketed.
    struct ProfClass {
        double ms = 0.0, bytes = 0.0;
        long samples = 0;
    };
    struct Pending {
        int cls;
        double bytes;
        long iter;
        cudaEvent_t a, b;
        long nl;  // launches in the sample (iterations iter .. iter + nl - 1)
    };
    bool prof = false;
    ProfClass pc[8];
    std::vector<cudaEvent_t> evpool;
    size_t evnext = 0;
    std::vector<Pending> pend;
    cudaEvent_t next_event() {
        if (evnext == evpool.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            evpool.push_back(e);
        }
        return evpool[evnext++];
    }
    cudaEvent_t prof_start() {
        cudaEvent_t a = next_event();
        CK(cudaEventRecord(a, s));
        return a;
    }
    void prof_stop(cudaEvent_t a, int cls, double bytes, long iter, long nl = 1) {
        cudaEvent_t b = next_event();
        CK(cudaEventRecord(b, s));
        pend.push_back(Pending{cls, bytes * nl, iter, a, b, nl});
    }
    // after a sync: keep samples of iterations that really executed
    void prof_flush(long executed) {
        for (auto& q : pend) {
            if (q.iter + q.nl > executed) continue;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, q.a, q.b));
            pc[q.cls].ms += ms;
            pc[q.cls].bytes += q.bytes;
            pc[q.cls].samples += q.nl;
        }
        pend.clear();
        evnext = 0;
    }

    void init(int dev) {
        device = dev;
        CK(cudaSetDevice(dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        partials.ensure(sizeof(double) * 1024 * 1024);
        counter.ensure(sizeof(unsigned) * 16);
        CK(cudaMemset(counter.p, 0, counter.bytes));
        scal.ensure(sizeof(double) * 16 * 8192);  // 16 scratch slots (sc(k))
        cgst.ensure(sizeof(CGState));
        hist.ensure(sizeof(double) * hist_cap);
        CK(cudaMallocHost(&st_host, 2 * sizeof(CGState)));
        for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : mark) CK(cudaEventCreate(&e));
    }
    ~Ctx() {
        if (s) cudaStreamSynchronize(s);
        for (auto& e : evpool) cudaEventDestroy(e);
        if (st_host) cudaFreeHost(st_host);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : mark)
            if (e) cudaEventDestroy(e);
        if (s) cudaStreamDestroy(s);
    }
    GridRed red() const { return GridRed{partials.template as<double>(), counter.template as<unsigned>()}; }
    // small device scratch: slot k of 8 slots of 8192 doubles
    double* sc(int k) const { return scal.template as<double>() + (size_t)k * 8192; }
    int grid_for(long n, int per = 256, int mult = 4) const {
        const long b = (n + per - 1) / per;
        return (int)std::max(1L, std::min<long>(b, (long)sms * mult));
    }
    void check_launch() {
        ++launches;
        CK(cudaGetLastError());
    }
    void sync() { CK(cudaStreamSynchronize(s)); }
};

// ------------------------------------------------------------ operator ---
struct DevOp {
    Ctx* ctx = nullptr;
    OpDev d{};
    DevBuf D, mu, F, Fpad;
    bool have_fields = false;
    double lam_max = 0.0;
    long n() const { return d.n; }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                   &q));
        if (!encode) throw CudaError("cuTensorMapEncodeTiled unavailable");
    }
    return encode;
}

// ------------------------------------------------------ launch helpers ---
inline dim3 stencil_grid(const OpDev& op, long zmult) {
    return dim3((unsigned)((op.N0 + 31) / 32), (unsigned)((op.N1 + 7) / 8), (unsigned)(op.N2 * zmult));
}

// z-chunk length: enough (i, j, k-chunk) blocks per column to fill the GPU
inline int stencil_kz(const OpDev& op, long ncols, int sms) {
    const long xy = (long)((op.N0 + 31) / 32) * ((op.N1 + 7) / 8);
    int kz = 1;
    while (kz < op.N2 && xy * ncols * ((op.N2 + 2 * kz - 1) / (2 * kz)) >= 8L * sms) kz *= 2;
    return kz;
}

// ---- multi-column stencil through TMA-staged planes (stencil_tma.cuh) ----
template <class T> CUtensorMap make_stencil_xmap(const OpDev& op, const T* x, long ldx, long xcols) {
    constexpr int W = Sc<T>::W;
    CUtensorMap m;
    cuuint64_t gdim[4] = {(cuuint64_t)op.N0 * W, (cuuint64_t)op.N1, (cuuint64_t)op.N2, (cuuint64_t)xcols};
    cuuint64_t gstride[3] = {(cuuint64_t)op.N0 * sizeof(T), (cuuint64_t)op.N0 * op.N1 * sizeof(T),
                             (cuuint64_t)ldx * sizeof(T)};
    cuuint32_t box[4] = {(cuuint32_t)(StX<T>::W * W), (cuuint32_t)SYH, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = tmap_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<T*>(x), gdim, gstride, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("stencil x tensor map: cuTensorMapEncodeTiled failed " + std::to_string((int)r));
    return m;
}
inline CUtensorMap make_stencil_fmap(const OpDev& op) {
    CUtensorMap m;
    const cuuint64_t rows = (cuuint64_t)op.N1 * op.N2;
    cuuint64_t gdim[4] = {(cuuint64_t)op.N0, (cuuint64_t)op.N1, (cuuint64_t)op.N2, 4};
    cuuint64_t gstride[3] = {(cuuint64_t)op.ldF * 8, (cuuint64_t)op.ldF * op.N1 * 8, (cuuint64_t)op.ldF * rows * 8};
    cuuint32_t box[4] = {(cuuint32_t)SFW, (cuuint32_t)SYH, 1, 4};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = tmap_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(op.Fp), gdim, gstride,
                               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("stencil field tensor map: cuTensorMapEncodeTiled failed " + std::to_string((int)r));
    return m;
}

// TMA strides / base must be 16-byte aligned: always for complex128; for
// float64 the x rows need an even N0 and an even column pitch.
template <class T> bool stencil_tma_ok(const OpDev& op, const T* x, long ldx) {
    static const int on = [] {
        const char* e = std::getenv("ROMDOT_STENCIL_TMA");
        return e ? std::atoi(e) : 1;
    }();
    if (!on || !op.Fp) return false;
    if (((uintptr_t)x & 15u) != 0) return false;
    if (sizeof(T) == 8 && (op.N0 % 2 != 0 || ldx % 2 != 0)) return false;
    return true;
}

template <class T, int NC, bool D2>
void launch_stencil_tma(Ctx& c, const OpDev& op, const T* x, long ldx, const int* xcol, T* y, long ldy, long ncols) {
    static const int S = [] {  // ring depth (2 planes resident, S - 2 in flight); 3..8, <= 227 KB
        const char* e = std::getenv("ROMDOT_STENCIL_STAGES");
        const int want = e ? std::max(3, std::min(8, std::atoi(e))) : 3;  // 3: two CTAs per SM (C5 sweep, profiles/r02_c5_stencil_sweep.jsonl)
        return std::min<int>(want, (int)(227 * 1024 / StTma<T>::stage(NC)));
    }();
    const size_t smem = (size_t)S * StTma<T>::stage(NC);
    static bool configured = false;
    if (!configured) {
        CK(cudaFuncSetAttribute(stencil_tma<T, NC, D2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    const CUtensorMap xm = make_stencil_xmap<T>(op, x, ldx, xcol ? (1L << 24) : ncols);
    const CUtensorMap fm = make_stencil_fmap(op);
    // marched units: planes (3D, grid over (i, j) tiles) or 8-row tiles (2D, grid over i tiles)
    const long bxy = (long)((op.N0 + SX - 1) / SX) * (D2 ? 1 : (op.N1 + SY - 1) / SY);
    const int nk = D2 ? (op.N1 + SY - 1) / SY : op.N2;
    const long groups = (ncols + NC - 1) / NC;
    // chunk length: as long as possible (3D plane re-loads at chunk seams cost
    // 2 / kz) while the grid still covers every SM a few times
    int kz = nk;
    while (kz > 8 && bxy * groups * ((nk + kz - 1) / kz) < 4L * c.sms) kz = (kz + 1) / 2;
    const long nkc = (nk + kz - 1) / kz;
    const long maxg = std::max(1L, 65535L / nkc);
    for (long g0 = 0; g0 < groups; g0 += maxg) {
        const long ng = std::min(maxg, groups - g0);
        const long cc0 = g0 * NC;
        const long nc = std::min(ng * NC, ncols - cc0);
        dim3 grid((unsigned)((op.N0 + SX - 1) / SX), (unsigned)(D2 ? 1 : (op.N1 + SY - 1) / SY), (unsigned)(nkc * ng));
        // column offsets go through the tensor-map coordinate (base stays aligned);
        // gathered columns through xcol
        if (xcol) {
            stencil_tma<T, NC, D2><<<grid, ST_THREADS, smem, c.s>>>(xm, fm, op, xcol + cc0, y + (size_t)cc0 * ldy,
                                                                     ldy, (int)nc, kz, S);
        } else {
            const CUtensorMap xo = cc0 ? make_stencil_xmap<T>(op, x + (size_t)cc0 * ldx, ldx, nc) : xm;
            stencil_tma<T, NC, D2><<<grid, ST_THREADS, smem, c.s>>>(xo, fm, op, nullptr, y + (size_t)cc0 * ldy,
                                                                     ldy, (int)nc, kz, S);
        }
        c.check_launch();
    }
}

template <class T> void launch_stencil(Ctx& c, const OpDev& op, const T* x, long ldx, const int* xcol, T* y,
                                       long ldy, long ncols) {
    if (ncols <= 0) return;
    if (ncols >= 2 && stencil_tma_ok<T>(op, x, ldx)) {
        constexpr int NC = Sc<T>::W == 2 ? 4 : 8;
        if (op.d == 2)
            launch_stencil_tma<T, NC, true>(c, op, x, ldx, xcol, y, ldy, ncols);
        else
            launch_stencil_tma<T, NC, false>(c, op, x, ldx, xcol, y, ldy, ncols);
        return;
    }
    static const int mc = [] {
        // opt-in: C5 sweep at 8 columns 2D f64 0.38 -> 0.62 of peak, but 3D c128
        // 0.50 -> 0.41 (fewer z-march blocks in flight); C4 refresh unchanged
        const char* e = std::getenv("ROMDOT_STENCIL_MC");
        return e ? std::atoi(e) : 0;
    }();
    if (mc && ncols >= 2) {  // coefficients once per node for 4 columns
        constexpr int NC = 4;
        const long groups = (ncols + NC - 1) / NC;
        const int kz = stencil_kz(op, groups, c.sms);
        const long nkc = (op.N2 + kz - 1) / kz;
        const long maxg = std::max(1L, 65535L / nkc);
        for (long g0 = 0; g0 < groups; g0 += maxg) {
            const long ng = std::min(maxg, groups - g0);
            const long c0 = g0 * NC;
            const long nc = std::min(ng * NC, ncols - c0);
            dim3 grid((unsigned)((op.N0 + 31) / 32), (unsigned)((op.N1 + 7) / 8), (unsigned)(nkc * ng));
            stencil_kernel_mc<T, NC><<<grid, 256, 0, c.s>>>(op, xcol ? x : x + (size_t)c0 * ldx, ldx,
                                                            xcol ? xcol + c0 : nullptr, y + (size_t)c0 * ldy, ldy,
                                                            (int)nc, kz);
            c.check_launch();
        }
        return;
    }
    const int kz = stencil_kz(op, ncols, c.sms);
    const long nkc = (op.N2 + kz - 1) / kz;
    const long maxc = std::max(1L, 65535L / nkc);
    for (long c0 = 0; c0 < ncols; c0 += maxc) {
        const long nc = std::min(maxc, ncols - c0);
        dim3 grid((unsigned)((op.N0 + 31) / 32), (unsigned)((op.N1 + 7) / 8), (unsigned)(nkc * nc));
        stencil_kernel<T><<<grid, 256, 0, c.s>>>(op, xcol ? x : x + (size_t)c0 * ldx, ldx, xcol ? xcol + c0 : nullptr,
                                                 y + (size_t)c0 * ldy, ldy, (int)nc, kz);
        c.check_launch();
    }
}

template <class T, bool HERM, int CPW, bool RB = false>
void ts_T_inst(Ctx& c, const T* K, long ldk, int cc, int col0, const T* x, long n, double* out, const CGState* st) {
    const long ntiles = (n + 32 * TSU<T, CPW>::U - 1) / (32 * TSU<T, CPW>::U);
    const int grid = (int)std::max(1L, std::min<long>(ntiles, (long)c.sms * 4));
    ts_T<T, HERM, CPW, RB><<<grid, TS_THREADS, 0, c.s>>>(K, ldk, cc, col0, x, n, c.red(), out, st);
    c.check_launch();
}

// out[j] = sum_i op(K_ij) x_i, j < ncol  (chunks of 128 columns). RB: row-blocked K (ldk = C).
template <class T, bool HERM, bool RB = false>
void ts_T_launch(Ctx& c, const T* K, long ldk, long ncol, const T* x, long n, double* out, const CGState* st = nullptr) {
    for (long col0 = 0; col0 < ncol; col0 += 128) {
        const int cc = (int)std::min(128L, ncol - col0);
        const int cpw = (cc + 7) / 8;
        if (cpw <= 1)
            ts_T_inst<T, HERM, 1, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
        else if (cpw <= 2)
            ts_T_inst<T, HERM, 2, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
        else if (cpw <= 4)
            ts_T_inst<T, HERM, 4, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
        else if (cpw <= 6)
            ts_T_inst<T, HERM, 6, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
        else if (cpw <= 8)
            ts_T_inst<T, HERM, 8, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
        else if (cpw <= 12)
            ts_T_inst<T, HERM, 12, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
        else
            ts_T_inst<T, HERM, 16, RB>(c, K, ldk, cc, (int)col0, x, n, out, st);
    }
}

template <class T, bool HERM, int CPW, bool RB = false>
void ts_NT_inst(Ctx& c, const T* K, long ldk, int cc, const T* x, T* xo, long n, const double* cin, double* out,
                const CGState* st) {
    const long ntiles = (n + 32 * TSU<T, CPW>::U - 1) / (32 * TSU<T, CPW>::U);
    const int grid = (int)std::max(1L, std::min<long>(ntiles, (long)c.sms * 2));
    ts_NT<T, HERM, CPW, RB><<<grid, TS_THREADS, 0, c.s>>>(K, ldk, cc, x, xo, n, cin, c.red(), out, st);
    c.check_launch();
}

template <class T>
void ts_N_launch(Ctx& c, const T* K, long ldk, long ncol, const T* x, T* xo, long n, const double* cin,
                 double csign = 1.0, const CGState* st = nullptr) {
    const size_t smem = sizeof(double) * Sc<T>::W * std::max(1L, ncol);
    if (smem > 48 * 1024) {
        // very wide bases: chunk columns (x - K[:, a:b] c[a:b] accumulated in xo)
        const T* src = x;
        for (long c0 = 0; c0 < ncol; c0 += 1024) {
            const long cc = std::min(1024L, ncol - c0);
            ts_N_launch<T>(c, K + (size_t)c0 * ldk, ldk, cc, src, xo, n, cin + (size_t)c0 * Sc<T>::W, csign, st);
            src = xo;
        }
        return;
    }
    ts_N<T><<<c.grid_for(n, 256, 8), 256, smem, c.s>>>(K, ldk, (int)ncol, x, xo, n, cin, csign, st);
    c.check_launch();
}

// fused {xo = x - K c1 ; out = op(K)^T xo} for ncol <= 128, else N then T
template <class T, bool HERM, bool RB = false>
void ts_NT_launch(Ctx& c, const T* K, long ldk, long ncol, const T* x, T* xo, long n, const double* cin,
                  double* out, const CGState* st = nullptr) {
    if (ncol > 128) {
        if (RB) throw ConfigError("row-blocked basis limited to 128 columns");
        ts_N_launch<T>(c, K, ldk, ncol, x, xo, n, cin, 1.0, st);
        ts_T_launch<T, HERM>(c, K, ldk, ncol, xo, n, out, st);
        return;
    }
    const int cc = (int)ncol;
    const int cpw = (cc + 7) / 8;
    if (cpw <= 1)
        ts_NT_inst<T, HERM, 1, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
    else if (cpw <= 2)
        ts_NT_inst<T, HERM, 2, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
    else if (cpw <= 4)
        ts_NT_inst<T, HERM, 4, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
    else if (cpw <= 6)
        ts_NT_inst<T, HERM, 6, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
    else if (cpw <= 8)
        ts_NT_inst<T, HERM, 8, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
    else if (cpw <= 12)
        ts_NT_inst<T, HERM, 12, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
    else
        ts_NT_inst<T, HERM, 16, RB>(c, K, ldk, cc, x, xo, n, cin, out, st);
}


// ------------------------------------------------ TMA projection launcher ---
constexpr long kRowPad = 256;  // row padding of RB bases and inner workspaces
inline long padded_rows(long n) { return (n + kRowPad - 1) / kRowPad * kRowPad; }

static CUtensorMap g_null_tmap;  // unused map passed to the 1D (row-blocked) variant

// Encode a 2D tensor map over a column-major n x ncols matrix (ld = n) viewed
// as doubles, box = 32 rows x bc columns (driver entry point, no -lcuda).
template <class T> CUtensorMap make_colmajor_tmap(const T* base, long n, long ld, long ncols, int bc) {
    auto encode = tmap_encode();
    constexpr int W = Sc<T>::W;
    CUtensorMap m;
    cuuint64_t gdim[2] = {(cuuint64_t)n * W, (cuuint64_t)ncols};
    cuuint64_t gstride[1] = {(cuuint64_t)ld * sizeof(T)};
    cuuint32_t box[2] = {(cuuint32_t)(32 * W), (cuuint32_t)bc};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<T*>(base), gdim, gstride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

template <class T, int MODE, int CPW>
void ts_tma_inst(Ctx& c, const T* Krb, int C, long n, const T* x, T* xo, const double* cin, double* out, T* r, T* p,
                 T* s, T* y, CGState* st, const T* G) {
    const int es = sizeof(T);
    const int NV = MODE == 2 ? 5 : 1;
    int TR = 256;
    while (TR > 32 && (long)TR * C * es > 48 * 1024) TR >>= 1;
    TmaLayout L = tma_layout<T>(C, TR, 2, NV);
    const uint32_t per_stage = ((L.tile_bytes + 127u) & ~127u) + NV * ((L.x_bytes + 127u) & ~127u);
    const uint32_t fixed = L.total - 2 * per_stage;
    int S = (int)std::min<long>(8, (196L * 1024 - fixed) / per_stage);
    if (S < 2) S = 2;
    L = tma_layout<T>(C, TR, S, NV);
    static int configured = 0;
    if (!configured) {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, ts_tma<T, MODE, false, CPW, false>));
        CK(cudaFuncSetAttribute(ts_tma<T, MODE, false, CPW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes));
        configured = optin - (int)fa.sharedSizeBytes;
    }
    if ((int)L.total > configured) throw ConfigError("TMA projection: shared-memory ring too large");
    const long ntile = padded_rows(n) / TR;
    const int grid = (int)std::max(1L, std::min<long>(ntile, (long)c.sms));
    ts_tma<T, MODE, false, CPW, false><<<grid, TMA_THREADS, L.total, c.s>>>(g_null_tmap, 0, Krb, C, n, ntile, L, x,
                                                                            xo, cin, c.red(), out, r, p, s, y, st, G);
    c.check_launch();
}

template <class T, int MODE>
void ts_tma_launch(Ctx& c, const T* Krb, int C, long n, const T* x, T* xo, const double* cin, double* out,
                   T* r = nullptr, T* p = nullptr, T* s = nullptr, T* y = nullptr, CGState* st = nullptr,
                   const T* G = nullptr) {
    if (C > 128) throw ConfigError("TMA projection limited to 128 columns");
    const int cpw = (C + 7) / 8;
    if (cpw <= 1)
        ts_tma_inst<T, MODE, 1>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else if (cpw <= 2)
        ts_tma_inst<T, MODE, 2>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else if (cpw <= 4)
        ts_tma_inst<T, MODE, 4>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else if (cpw <= 6)
        ts_tma_inst<T, MODE, 6>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else if (cpw <= 8)
        ts_tma_inst<T, MODE, 8>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else if (cpw <= 10)
        ts_tma_inst<T, MODE, 10>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else if (cpw <= 12)
        ts_tma_inst<T, MODE, 12>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
    else
        ts_tma_inst<T, MODE, 16>(c, Krb, C, n, x, xo, cin, out, r, p, s, y, st, G);
}

// ------------------------------------------------- fused CG iteration launcher ---
// cg_fused (cg_fused.cuh): update of iteration i + stencil, dots and K^T w of
// iteration i+1 in one launch, one HBM stream of the row-blocked K.
template <class T, int CPW>
void cg_fused_inst(Ctx& c, const OpDev& op, const T* Krb, int C, T* w, T* r, T* p, T* s, T* y, CGState* st,
                   double* cbuf, const T* G) {
    const long n = op.n;
    const int es = sizeof(T);
    int TR = 256;
    while (TR > 32 && (long)TR * C * es > 48 * 1024) TR >>= 1;
    FusedLayout L = fused_layout<T>(C, TR, 2);
    const uint32_t fixed = L.total - 2 * L.stage_bytes;
    static const long cap_kb = [] {
        const char* e = std::getenv("ROMDOT_FUSED_SMEM_KB");
        return e ? std::atol(e) : 222L;
    }();
    int S = (int)std::min<long>(8, (cap_kb * 1024 - fixed) / L.stage_bytes);
    if (S < 2) S = 2;
    L = fused_layout<T>(C, TR, S);
    static int configured = 0;
    if (!configured) {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, cg_fused<T, CPW>));
        CK(cudaFuncSetAttribute(cg_fused<T, CPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes));
        configured = optin - (int)fa.sharedSizeBytes;
    }
    if ((int)L.total > configured) throw ConfigError("fused CG iteration: shared-memory ring too large");
    const long ntile = padded_rows(n) / TR;
    const int grid = (int)std::max(1L, std::min<long>(ntile, (long)c.sms));
    const long P = op.d == 3 ? (long)op.N0 * op.N1 : (long)op.N0;
    const long D = (TR - 1 + P) / TR;
    L.L = (int)((grid - 1 + D) / grid);
    static const int slack = [] {
        const char* e = std::getenv("ROMDOT_FUSED_SLACK");
        return e ? std::max(0, std::atoi(e)) : 7;
    }();
    L.LI = L.L + slack;
    static const int pf = [] {
        const char* e = std::getenv("ROMDOT_FUSED_PF");
        return e ? std::max(0, std::atoi(e)) : 0;
    }();
    L.PF = pf;
    static const int poll_ns = [] {
        const char* e = std::getenv("ROMDOT_FUSED_POLL_NS");
        return e ? std::max(0, std::atoi(e)) : 2000;  // ns; 64 measured 10% slower (power: the polls keep the GPU at its 1000 W cap)
    }();
    L.poll_ns = poll_ns;
    static const int rel_ns = [] {
        const char* e = std::getenv("ROMDOT_FUSED_REL_NS");
        return e ? std::max(0, std::atoi(e)) : 256;
    }();
    L.rel_ns = rel_ns;
    static const int ahead = [] {
        const char* e = std::getenv("ROMDOT_FUSED_AHEAD");
        return e ? std::atoi(e) : 1;
    }();
    L.ahead = ahead;
    static const int relbatch = [] {
        const char* e = std::getenv("ROMDOT_FUSED_RELBATCH");
        return e ? std::atoi(e) : 1;
    }();
    L.relbatch = relbatch;
    static const int dbg = [] {
        const char* e = std::getenv("ROMDOT_FUSED_DBG");
        return e ? std::atoi(e) : 0;
    }();
    L.dbg = dbg;
    const long nsteps = (ntile + grid - 1) / grid;
    if (c.fstep.bytes < sizeof(unsigned) * nsteps) {
        c.fstep.ensure(sizeof(unsigned) * (nsteps + 1024));
        CK(cudaMemsetAsync(c.fstep.p, 0, c.fstep.bytes, c.s));
    }
    static const bool tprof = [] {
        const char* e = std::getenv("ROMDOT_FUSED_PROF");
        return e && std::atoi(e) != 0;
    }();
    if (tprof && !c.fprof.p) {
        c.fprof.ensure(sizeof(unsigned long long) * 56);  // 5 roles x 8 slots + launch phases
        c.fprof_reset();
    }
    static const bool pdl = [] {
        // opt-in: 5.8 -> 3.6 us between launches, but the fixed-length probe's
        // wall time per iteration got 2-5x worse with it (not understood yet)
        const char* e = std::getenv("ROMDOT_FUSED_PDL");
        return e ? std::atoi(e) != 0 : false;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(FU_THREADS);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = c.s;
    // Cooperative launch: the CTAs spin on one another's step counters, so they
    // must all be resident at once. The attribute makes the driver guarantee
    // that (or fail the launch with cudaErrorCooperativeLaunchTooLarge, e.g.
    // when another kernel or MPS client holds SMs) instead of hanging.
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    static const bool fcheck = [] {
        const char* e = std::getenv("ROMDOT_FUSED_CHECK");
        return e && std::atoi(e) != 0;
    }();
    unsigned* chk = nullptr;
    if (fcheck) {
        const size_t need = sizeof(unsigned) * (16 + ntile + 256);
        if (c.fchk.bytes < need) {
            c.fchk.ensure(need);
            CK(cudaMemsetAsync(c.fchk.p, 0, c.fchk.bytes, c.s));
        }
        chk = c.fchk.template as<unsigned>();
    }
    CK(cudaLaunchKernelEx(&cfg, cg_fused<T, CPW>, op, Krb, C, ntile, L, w, r, p, s, y, st,
                          c.hist.template as<double>(), c.red(), cbuf, c.fstep.template as<unsigned>(), G,
                          tprof ? c.fprof.template as<unsigned long long>() : (unsigned long long*)nullptr, chk,
                          ++c.fchk_epoch));
    if (tprof) ++c.fprof_launches;
    c.check_launch();
}

template <class T>
void cg_fused_launch(Ctx& c, const OpDev& op, const T* Krb, int C, T* w, T* r, T* p, T* s, T* y, CGState* st,
                     double* cbuf, const T* G) {
    if (C > 128 || C < 1) throw ConfigError("fused CG iteration: 1..128 recycle columns");
    const int cpw = (C + 7) / 8;
    if (cpw <= 1)
        cg_fused_inst<T, 1>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else if (cpw <= 2)
        cg_fused_inst<T, 2>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else if (cpw <= 4)
        cg_fused_inst<T, 4>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else if (cpw <= 6)
        cg_fused_inst<T, 6>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else if (cpw <= 8)
        cg_fused_inst<T, 8>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else if (cpw <= 10)
        cg_fused_inst<T, 10>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else if (cpw <= 12)
        cg_fused_inst<T, 12>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
    else
        cg_fused_inst<T, 16>(c, op, Krb, C, w, r, p, s, y, st, cbuf, G);
}

// nrm[0] = ||x||^2, nrm[1..W] = x^T x
template <class T> void launch_norms(Ctx& c, const T* x, long n, double* nrm) {
    vec_norms<T><<<c.grid_for(n, 256, 2), 256, 0, c.s>>>(x, n, c.red(), nrm);
    c.check_launch();
}

template <class T> void launch_scale(Ctx& c, const T* x, T* y, long n, const double* nrm, int mode) {
    vec_scale_by_rho<T><<<c.grid_for(n, 256, 8), 256, 0, c.s>>>(x, y, n, nrm, mode);
    c.check_launch();
}

inline void launch_addsub(Ctx& c, int m, const double* a, const double* b, double sgn, double* out) {
    if (m <= 0) return;
    dvec_addsub<<<(m + 255) / 256, 256, 0, c.s>>>(m, a, b, sgn, out);
    c.check_launch();
}

// CGS2 of z against the first t columns of Q (op = H or T): q = (I - QQ^op)^2 z,
// coef (device, t scalars) = Q^op z accumulated over both passes.
template <class T, bool HERM>
void cgs2(Ctx& c, const T* Q, long ldq, long t, const T* z, T* q, long n, double* coef, double* tmp1,
          double* tmp2) {
    constexpr int W = Sc<T>::W;
    if (t == 0) {
        if (q != z) CK(cudaMemcpyAsync(q, z, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        return;
    }
    ts_T_launch<T, HERM>(c, Q, ldq, t, z, n, tmp1);
    ts_NT_launch<T, HERM>(c, Q, ldq, t, z, q, n, tmp1, tmp2);
    ts_N_launch<T>(c, Q, ldq, t, q, q, n, tmp2);
    launch_addsub(c, (int)(t * W), tmp1, tmp2, 1.0, coef);
}


// ------------------------------------------------------- block helpers ---
// G (a x b, device, ld a) = op(X)^T Y over n rows. sym: X == Y, upper tiles only.
template <class T, bool HERM, int B, int CPW>
void gram_thin_launch(Ctx& c, const T* X, long ldx, long a, const T* Y, long ldy, long b, long n, T* G) {
    const long chunks = (a + 8 * CPW - 1) / (8 * CPW);
    static int per_sm = 0;
    if (!per_sm) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gram_thin<T, HERM, B, CPW>, 256, 0));
        per_sm = std::max(1, per_sm);
    }
    const long want = std::max(1L, (long)c.sms * std::max(1, per_sm) / chunks);
    const int gx = (int)std::max(1L, std::min<long>((n + 31) / 32, want));
    if ((long)gx * chunks * 8 * CPW * B * Sc<T>::W > 1024L * 1024) throw ConfigError("gram_thin: partials");
    dim3 grid(gx, (unsigned)chunks);
    gram_thin<T, HERM, B, CPW><<<grid, 256, 0, c.s>>>(X, ldx, (int)a, Y, ldy, (int)b, n, c.red(), G);
    c.check_launch();
}

// pipelined thin Gram: one CTA per SM, NS-stage cp.async ring of RT-row tiles
template <class T, bool HERM, int B, int CPW, int RT>
void gram_thin_pipe_launch(Ctx& c, const T* X, long ldx, long a, const T* Y, long ldy, long b, long n, T* G) {
    constexpr int NC = 8 * CPW;
    constexpr size_t stage = sizeof(T) * (NC + B) * RT;
    constexpr int NS = stage * 6 <= 210 * 1024 ? 6 : (stage * 5 <= 210 * 1024 ? 5 : (stage * 4 <= 210 * 1024 ? 4 : 3));
    constexpr size_t smem = stage * NS;
    static_assert(smem <= 220 * 1024, "gram_thin_pipe: ring too large");
    static bool configured = false;
    if (!configured) {
        CK(cudaFuncSetAttribute(gram_thin_pipe<T, HERM, B, CPW, NS, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        configured = true;
    }
    const long chunks = (a + NC - 1) / NC;
    const int gx = (int)std::max(1L, std::min<long>((n + RT - 1) / RT, (long)c.sms));
    if ((long)gx * chunks * NC * B * Sc<T>::W > 1024L * 1024) throw ConfigError("gram_thin: partials");
    dim3 grid(gx, (unsigned)chunks);
    gram_thin_pipe<T, HERM, B, CPW, NS, RT><<<grid, 256, smem, c.s>>>(X, ldx, (int)a, Y, ldy, (int)b, n, c.red(), G);
    c.check_launch();
}

template <class T, bool HERM, int B, int CPW>
void gram_thin_pipe_rt(Ctx& c, const T* X, long ldx, long a, const T* Y, long ldy, long b, long n, T* G) {
    static const int rt = [] {
        const char* e = std::getenv("ROMDOT_GRAM_THIN_RT");
        return e ? std::atoi(e) : 64;
    }();
    if constexpr (CPW <= 8) {
        if (rt == 64) {
            gram_thin_pipe_launch<T, HERM, B, CPW, 64>(c, X, ldx, a, Y, ldy, b, n, G);
            return;
        }
    }
    gram_thin_pipe_launch<T, HERM, B, CPW, 32>(c, X, ldx, a, Y, ldy, b, n, G);
}

// columns per warp: one block row over all a columns when the accumulators fit
// (ROMDOT_GRAM_THIN=0 keeps the register-staged kernel)
template <class T, bool HERM, int B>
void gram_thin_cpw(Ctx& c, const T* X, long ldx, long a, const T* Y, long ldy, long b, long n, T* G) {
    static const int pipe = [] {
        const char* e = std::getenv("ROMDOT_GRAM_THIN");
        return e ? std::atoi(e) : 1;
    }();
    if constexpr (B <= 4) {
        // measured at n = 2M complex (exp: a = 64 / 69 / 81, b = 4): 0.48 / 0.71 / 0.71
        // ms against 0.60 / 0.88 / 0.89 for the register-staged kernel, which
        // stays faster for small L2-resident real problems (C3: n = 262k)
        if (pipe && a <= 96 && n >= (1L << 20)) {
            if (a <= 32)
                gram_thin_pipe_rt<T, HERM, B, 4>(c, X, ldx, a, Y, ldy, b, n, G);
            else if (a <= 64)
                gram_thin_pipe_rt<T, HERM, B, 8>(c, X, ldx, a, Y, ldy, b, n, G);
            else
                gram_thin_pipe_rt<T, HERM, B, 12>(c, X, ldx, a, Y, ldy, b, n, G);
            return;
        }
    }
    gram_thin_launch<T, HERM, B, 4>(c, X, ldx, a, Y, ldy, b, n, G);
}

template <class T, bool HERM>
void gram(Ctx& c, const T* X, long ldx, long a, const T* Y, long ldy, long b, long n, T* G, bool sym, DevBuf& work) {
    if (a == 0 || b == 0) return;
    if (!sym && b <= 8 && a <= 256) {  // thin: multi-vector T pass (no wasted tile FLOPs)
        if (b <= 2)
            gram_thin_cpw<T, HERM, 2>(c, X, ldx, a, Y, ldy, b, n, G);
        else if (b <= 4)
            gram_thin_cpw<T, HERM, 4>(c, X, ldx, a, Y, ldy, b, n, G);
        else
            gram_thin_cpw<T, HERM, 8>(c, X, ldx, a, Y, ldy, b, n, G);
        return;
    }
    const long ta = (a + GT<T>::TA - 1) / GT<T>::TA, tb = (b + GT<T>::TB - 1) / GT<T>::TB;
    const long tiles = sym ? ta * (ta + 1) / 2 : ta * tb;
    long slices = std::max(1L, std::min<long>((4L * c.sms + tiles - 1) / tiles, (n + 4095) / 4096));
    slices = std::min(slices, 1024L);
    long rps = (n + slices - 1) / slices;
    rps = (rps + GT<T>::KC - 1) / GT<T>::KC * GT<T>::KC;
    slices = (n + rps - 1) / rps;
    work.ensure(sizeof(T) * slices * a * b);
    dim3 grid((unsigned)ta, (unsigned)tb, (unsigned)slices);
    gram_kernel<T, HERM><<<grid, GT<T>::THREADS, 0, c.s>>>(X, ldx, (int)a, Y, ldy, (int)b, n, rps,
                                                            work.template as<T>(), sym);
    c.check_launch();
    gram_reduce<T, HERM><<<c.grid_for(a * b, 256, 4), 256, 0, c.s>>>(work.template as<T>(), (int)slices, (int)a,
                                                                      (int)b, G, sym);
    c.check_launch();
}

// Z = X M (SUB=false) or Z = Y - X M (SUB=true); M is a x b on the device (ld a).
template <class T, int B>
void gemm_thin_launch(Ctx& c, const T* X, long ldx, long a, const T* M, long b, const T* Y, long ldy, T* Z, long ldz,
                      long n) {
    gemm_thin_sub<T, B><<<c.grid_for(n, 256, 8), 256, sizeof(T) * a * b, c.s>>>(X, ldx, (int)a, M, (int)b, Y, ldy, Z,
                                                                              ldz, n);
    c.check_launch();
}

template <class T, bool SUB>
void gemm(Ctx& c, const T* X, long ldx, long a, const T* M, long b, const T* Y, long ldy, T* Z, long ldz, long n,
          bool upper) {
    if (b == 0 || n == 0) return;
    if (SUB && a > 0 && b <= 8 && sizeof(T) * a * b <= 48 * 1024) {  // thin: thread-per-row N pass
        if (b <= 2)
            gemm_thin_launch<T, 2>(c, X, ldx, a, M, b, Y, ldy, Z, ldz, n);
        else if (b <= 4)
            gemm_thin_launch<T, 4>(c, X, ldx, a, M, b, Y, ldy, Z, ldz, n);
        else
            gemm_thin_launch<T, 8>(c, X, ldx, a, M, b, Y, ldy, Z, ldz, n);
        return;
    }
    if (a == 0) {
        if (SUB && Z != Y)
            for (long j = 0; j < b; ++j)
                CK(cudaMemcpyAsync(Z + j * ldz, Y + j * ldy, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        return;
    }
    static const int dmma_on = [] {
        const char* e = std::getenv("ROMDOT_GEMM_DMMA");
        return e ? std::atoi(e) : 1;
    }();
    if (dmma_on && a >= 32) {  // FP64 tensor cores (gemm_tall_dmma); DFMA kernel below otherwise
        constexpr int TCD = GDT<T>::TC;
        constexpr size_t smem = gemm_dmma_smem<T>();
        static bool configured = false;
        if (!configured) {
            CK(cudaFuncSetAttribute(gemm_tall_dmma<T, SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            configured = true;
        }
        const long rtd = (n + GD_TR - 1) / GD_TR;
        for (long r0 = 0; r0 < rtd; r0 += 65535) {
            const long nr = std::min(65535L, rtd - r0);
            const long off = r0 * GD_TR;
            dim3 grid((unsigned)((b + TCD - 1) / TCD), (unsigned)nr);
            gemm_tall_dmma<T, SUB><<<grid, 256, smem, c.s>>>(X + off, ldx, (int)a, M, (int)b, SUB ? Y + off : nullptr,
                                                          ldy, Z + off, ldz, std::min(n - off, nr * GD_TR), upper);
            c.check_launch();
        }
        return;
    }
    constexpr int TC = Sc<T>::W == 1 ? 64 : 32;
    const long rt = (n + 63) / 64;
    for (long r0 = 0; r0 < rt; r0 += 65535) {
        const long nr = std::min(65535L, rt - r0);
        const long off = r0 * 64;
        dim3 grid((unsigned)((b + TC - 1) / TC), (unsigned)nr);
        gemm_tall<T, SUB><<<grid, 256, 0, c.s>>>(X + off, ldx, (int)a, M, (int)b, SUB ? Y + off : nullptr, ldy,
                                                  Z + off, ldz, std::min(n - off, nr * 64), upper);
        c.check_launch();
    }
}

// In-place upper Cholesky (HERM: S^H S, else S^T S) + inverse; returns the
// pivot diagnostics and the 1-norm condition estimate of S.
struct CholInfo {
    int bad = 0;
    double kappa1 = 0.0;
};
template <class T, bool HERM> CholInfo chol_inv(Ctx& c, T* G, T* Sinv, long r, bool want_kappa) {
    CholInfo ci;
    if (r == 0) return ci;
    double* info = c.sc(7) + 32;
    chol_upper<T, HERM><<<1, 1024, 0, c.s>>>(G, (int)r, info);
    c.check_launch();
    tri_inv_upper<T><<<1, 1024, 0, c.s>>>(G, Sinv, (int)r);
    c.check_launch();
    double hi[3];
    CK(cudaMemcpyAsync(hi, info, sizeof(hi), cudaMemcpyDeviceToHost, c.s));
    std::vector<T> S, Si;
    if (want_kappa) {
        S.resize(r * r);
        Si.resize(r * r);
        CK(cudaMemcpyAsync(S.data(), G, sizeof(T) * r * r, cudaMemcpyDeviceToHost, c.s));
        CK(cudaMemcpyAsync(Si.data(), Sinv, sizeof(T) * r * r, cudaMemcpyDeviceToHost, c.s));
    }
    c.sync();
    ci.bad = (int)hi[0];
    if (want_kappa) {
        double n1 = 0.0, n2 = 0.0;
        for (long j = 0; j < r; ++j) {
            double a = 0.0, b = 0.0;
            for (long i = 0; i <= j; ++i) {
                a += std::sqrt(Sc<T>::abs2(S[i + j * r]));
                b += std::sqrt(Sc<T>::abs2(Si[i + j * r]));
            }
            n1 = std::max(n1, a);
            n2 = std::max(n2, b);
        }
        ci.kappa1 = n1 * n2;
        if (!std::isfinite(ci.kappa1)) ci.bad = ci.bad ? ci.bad : 1;
    }
    return ci;
}


// ---- column-major (global basis) TMA passes, 128-column chunks -----------
// out[j] = sum_i op(K_ij) x_i (MODE 0) and xo = x - K c (MODE 3) over a
// column-major n x ncols matrix with ld*sizeof(T) % 16 == 0. x / xo must be
// padded to padded_rows(n) (the TMA x tile of the last row block).
template <class T, int MODE, bool HERM>
void global_tma_chunk(Ctx& c, const T* K, long ld, long ncols, long col0, int cc, const T* x, T* xo, const double* cin,
                      double* out, long n, CGState* st = nullptr) {
    constexpr int CPW = 16;
    const int es = sizeof(T);
    TmaLayout L = tma_layout<T>(cc, 32, 2, 1);
    const uint32_t per_stage = ((L.tile_bytes + 127u) & ~127u) + ((L.x_bytes + 127u) & ~127u);
    const uint32_t fixed = L.total - 2 * per_stage;
    int S = (int)std::min<long>(8, (196L * 1024 - fixed) / per_stage);
    if (S < 2) S = 2;
    L = tma_layout<T>(cc, 32, S, 1);
    static int configured = 0;
    if (!configured) {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, ts_tma<T, MODE, HERM, CPW, true>));
        CK(cudaFuncSetAttribute(ts_tma<T, MODE, HERM, CPW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes));
        configured = optin - (int)fa.sharedSizeBytes;
    }
    if ((int)L.total > configured) throw ConfigError("global TMA pass: shared-memory ring too large");
    const CUtensorMap tm = make_colmajor_tmap<T>(K, n, ld, ncols, cc);
    const long ntile = padded_rows(n) / 32;
    const int grid = (int)std::max(1L, std::min<long>(ntile, (long)c.sms));
    ts_tma<T, MODE, HERM, CPW, true><<<grid, TMA_THREADS, L.total, c.s>>>(
        tm, (int)col0, nullptr, cc, n, ntile, L, x, xo, cin ? cin + col0 * Sc<T>::W : nullptr, c.red(),
        out ? out + col0 * Sc<T>::W : nullptr, nullptr, nullptr, nullptr, nullptr, st, nullptr);
    c.check_launch();
    (void)es;
}

template <class T> bool tma_ok(long ld) {
    static const int off = [] {
        const char* e = std::getenv("ROMDOT_NO_GLOBAL_TMA");
        return e ? std::atoi(e) : 0;
    }();
    return !off && (ld * (long)sizeof(T)) % 16 == 0;
}

// out = op(K)^T x   (x padded)
template <class T, bool HERM>
void global_T(Ctx& c, const T* K, long ld, long ncols, const T* x, long n, double* out, CGState* st = nullptr) {
    if (!tma_ok<T>(ld)) {
        ts_T_launch<T, HERM>(c, K, ld, ncols, x, n, out, st);
        return;
    }
    for (long c0 = 0; c0 < ncols; c0 += 128)
        global_tma_chunk<T, 0, HERM>(c, K, ld, ncols, c0, (int)std::min(128L, ncols - c0), x, nullptr, nullptr, out, n,
                                     st);
}

// xo = x - K cin  (x, xo padded; may alias)
template <class T>
void global_N(Ctx& c, const T* K, long ld, long ncols, const T* x, T* xo, long n, const double* cin,
              CGState* st = nullptr) {
    if (!tma_ok<T>(ld) || ncols == 0) {
        ts_N_launch<T>(c, K, ld, ncols, x, xo, n, cin, 1.0, st);
        return;
    }
    const T* src = x;
    for (long c0 = 0; c0 < ncols; c0 += 128) {
        global_tma_chunk<T, 3, false>(c, K, ld, ncols, c0, (int)std::min(128L, ncols - c0), src, xo, cin, nullptr, n,
                                      st);
        src = xo;
    }
}

// CGS2 of z against the first t columns of Q with padded vectors (TMA path)
template <class T, bool HERM>
void cgs2_global(Ctx& c, const T* Q, long ldq, long t, const T* z, T* q, long n, double* coef, double* tmp1,
                 double* tmp2) {
    constexpr int W = Sc<T>::W;
    if (t == 0) {
        if (q != z) CK(cudaMemcpyAsync(q, z, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        return;
    }
    global_T<T, HERM>(c, Q, ldq, t, z, n, tmp1);
    global_N<T>(c, Q, ldq, t, z, q, n, tmp1);
    global_T<T, HERM>(c, Q, ldq, t, q, n, tmp2);
    global_N<T>(c, Q, ldq, t, q, q, n, tmp2);
    launch_addsub(c, (int)(t * W), tmp1, tmp2, 1.0, coef);
}

// CGS2 with the second pass run only when the first cancelled more than half
// of ||z||^2 (reorth_decide; device-side, no host sync). nrmz[0] = ||z||^2 on
// entry (launch_norms). flag is scratch device state.
template <class T, bool HERM>
void cgs2_global_selective(Ctx& c, const T* Q, long ldq, long t, const T* z, T* q, long n, double* coef,
                           double* tmp1, double* tmp2, const double* nrmz, CGState* flag) {
    constexpr int W = Sc<T>::W;
    if (t == 0) {
        if (q != z) CK(cudaMemcpyAsync(q, z, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        return;
    }
    global_T<T, HERM>(c, Q, ldq, t, z, n, tmp1);
    global_N<T>(c, Q, ldq, t, z, q, n, tmp1);
    double* nrmq = c.sc(8);
    launch_norms<T>(c, q, n, nrmq);
    reorth_decide<<<1, 256, 0, c.s>>>(nrmq, nrmz, (int)(t * W), tmp2, flag);
    c.check_launch();
    global_T<T, HERM>(c, Q, ldq, t, q, n, tmp2, flag);
    global_N<T>(c, Q, ldq, t, q, q, n, tmp2, flag);
    launch_addsub(c, (int)(t * W), tmp1, tmp2, 1.0, coef);
}

// ---------------------------------------------------------- CG driver ---
struct SolveOut {
    int iterations = 0;
    bool converged = false;
    double final_relres = 0.0;
    double correction_norm = 0.0;
    std::vector<double> hist;
};

// CholQR refresh: a second pass when the 1-norm condition estimate of the first
// pass's factor exceeds this (default 20; ROMDOT_REFRESH_KAPPA)
inline double refresh_kappa() {
    static const double k = [] {
        const char* e = std::getenv("ROMDOT_REFRESH_KAPPA");
        return e ? std::atof(e) : 20.0;
    }();
    return k;
}

template <class T> struct Workspace {
    DevBuf r, w, p, s, y, tmp, vec, krb, gk, gwork;
    void ensure(long n) {
        const size_t b = sizeof(T) * n;
        r.ensure(b);
        w.ensure(b);
        p.ensure(b);
        s.ensure(b);
        y.ensure(b);
        tmp.ensure(b);
        vec.ensure(b);
    }
};

// One-pass inner projection with the Gram-corrected second CGS coefficient
// (default; ROMDOT_CGS1G=0 selects the three-stream CGS2, ROMDOT_NO_TMA the
// non-TMA kernels, which use CGS2).
// Fused one-launch iteration (cg_fused.cuh) on top of the one-pass projection
// (default; ROMDOT_FUSED=0 keeps the three-launch iteration).
// Read per solve (not cached) so a test can compare both paths in one process.
inline bool use_fused_iteration() {
    const char* e = std::getenv("ROMDOT_FUSED");
    return (e ? std::atoi(e) : 1) != 0;
}

inline bool use_one_pass_projection() {
    static const bool on = [] {
        const char* e = std::getenv("ROMDOT_CGS1G");
        const char* t = std::getenv("ROMDOT_NO_TMA");
        return (e ? std::atoi(e) : 1) != 0 && (t ? std::atoi(t) : 0) == 0;
    }();
    return on;
}

// Recycled CG / COCG (the CPU checker under oracle/ restates the same recurrence).
// rhs, U, K, g, y_out, image: device. g/y_out/image may alias workspace-free
// buffers only.
// padded_io: rhs, y_out and image are zero-tailed to padded_rows(n), so the
// column-major U / K passes outside the iteration loop can use the TMA path.
template <class T>
SolveOut recycled_cg(Ctx& c, DevOp& op, const T* U, const T* K, long ncol, const T* rhs, double tol, long maxit,
                     double rhs_scale, T* g, T* y_out, T* image, Workspace<T>& ws, bool want_hist,
                     bool padded_io = false, const T* Gpre = nullptr) {
    constexpr int W = Sc<T>::W;
    const long n = op.n();
    const long npad = padded_rows(n);
    ws.ensure(npad);
    T* r = ws.r.template as<T>();
    T* w = ws.w.template as<T>();
    T* p = ws.p.template as<T>();
    T* s = ws.s.template as<T>();
    T* y = ws.y.template as<T>();
    double* e = c.sc(0);
    double* c1 = c.sc(1);
    double* c2 = c.sc(2);
    double* nrm = c.sc(3);
    if (ncol > 1024) throw ConfigError("recycle space wider than 1024 columns");
    CK(cudaMemsetAsync(r, 0, sizeof(T) * npad, c.s));
    CK(cudaMemsetAsync(w, 0, sizeof(T) * npad, c.s));
    // r0 = P rhs (CGS2), e = K^T rhs
    if (ncol > 0) {
        if (padded_io) {
            // selective second pass (Kahan-Parlett, device-side): 2 streams over K
            // instead of 4 when the first pass keeps at least half of ||rhs||^2
            launch_norms<T>(c, rhs, n, c.sc(3) + 8);
            c.rflag.ensure(sizeof(CGState));
            cgs2_global_selective<T, false>(c, K, n, ncol, rhs, r, n, e, c1, c2, c.sc(3) + 8,
                                            c.rflag.template as<CGState>());
        } else {
            cgs2<T, false>(c, K, n, ncol, rhs, r, n, e, c1, c2);
        }
    } else {
        CK(cudaMemcpyAsync(r, rhs, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
    }
    double scale = rhs_scale;
    if (!(scale > 0.0)) {
        launch_norms<T>(c, rhs, n, nrm);
        double h;
        CK(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        scale = std::sqrt(h);
    }
    CK(cudaMemsetAsync(y, 0, sizeof(T) * npad, c.s));
    CK(cudaMemsetAsync(p, 0, sizeof(T) * npad, c.s));
    CK(cudaMemsetAsync(s, 0, sizeof(T) * npad, c.s));
    CGState init{};
    init.scale = scale;
    init.tol = tol;
    init.maxit = (int)std::min<long>(maxit, 0x7fffffff);
    init.hist_cap = c.hist_cap;
    CGState* st = c.cgst.template as<CGState>();
    c.st_host[0] = init;
    CK(cudaMemcpyAsync(st, &c.st_host[0], sizeof(CGState), cudaMemcpyHostToDevice, c.s));
    CK(cudaStreamSynchronize(c.s));  // st_host slot reused below

    // stencil+dots: (32 x 8) x-y tiles marching over kz planes; the smallest kz
    // whose grid fits ONE resident wave (a partial second wave left the SMs 35%
    // idle at 128^3: ncu, 1.73 waves)
    dim3 grid_st = stencil_grid(op.d, 1);
    static int occ = 0;
    if (!occ) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cg_stencil_dots<T>, 256, 0));
        occ = std::max(1, occ);
    }
    const long wave = (long)occ * c.sms;
    int kz = 1;
    while ((long)grid_st.x * grid_st.y * ((op.d.N2 + kz - 1) / kz) > wave && kz < op.d.N2) ++kz;
    grid_st.z = (unsigned)((op.d.N2 + kz - 1) / kz);
    // row-blocked copy of K for the inner-iteration kernels (contiguous 32-row tiles)
    const T* Kit = K;
    if (ncol > 0) {
        if (sizeof(T) * npad * ncol > ws.krb.bytes) ws.krb.ensure(sizeof(T) * npad * (ncol + 16));  // slack
        repack_rb<T><<<c.grid_for(npad * ncol, 256, 8), 256, 0, c.s>>>(K, n, (int)ncol, n, ws.krb.template as<T>(),
                                                                      npad);
        c.check_launch();
        Kit = ws.krb.template as<T>();
    }
    const size_t smem_c = sizeof(double) * W * std::max(1L, ncol);
    // Default: one-pass projection with the Gram-corrected second CGS
    // coefficient, c2 = K^T (w - K c1) = c1 - G c1 with G = K^T K formed once
    // per solve -- two streams over K per iteration instead of three. Same
    // iteration counts and residuals as the three-stream CGS2 at C4 (29,206
    // iterations, max residual 9.98e-9 over three systems) in 24% less time.
    // ROMDOT_CGS1G=0 selects the three-stream CGS2 (MODE 0 / 1 / 2).
    const bool gram_pass = use_one_pass_projection() && ncol > 0 && ncol <= 128;
    const T* Gk = Gpre;
    if (gram_pass && !Gk) {
        ws.gk.ensure(sizeof(T) * ncol * ncol);
        gram<T, false>(c, K, n, ncol, K, n, ncol, n, ws.gk.template as<T>(), true, ws.gwork);
        Gk = ws.gk.template as<T>();
    }
    const int batch = n < 200000 ? 16 : 8;
    long batches = 0;
    const double es = sizeof(T);
    const bool fused = gram_pass && use_fused_iteration();
    cudaEvent_t fused_ev = nullptr;
    auto launch_batch = [&]() {
        for (int b = 0; b < batch; ++b) {
            const bool samp = c.prof && b == 0;
            const long iter = batches * batch;
            if (fused) {
                if (batches == 0 && b == 0) {
                    // head of iteration 0: w = A r0, dots, alpha_0 ; c1 = K^T w
                    cg_stencil_dots<T><<<grid_st, 256, 0, c.s>>>(op.d, r, w, st, c.hist.template as<double>(),
                                                                 c.red(), kz);
                    c.check_launch();
                    ts_tma_launch<T, 0>(c, Kit, (int)ncol, n, w, nullptr, nullptr, c1, nullptr, nullptr, nullptr,
                                        nullptr, st);
                } else {
                    // update of iteration i + head of iteration i+1, one stream of K.
                    // Sampled as a whole batch of back-to-back launches (an event
                    // pair around every launch adds ~20 us of front-end gap to it);
                    // kept only if all of them executed (prof_flush)
                    const bool bs = c.prof && batches > 0;
                    cudaEvent_t e4 = bs && b == 0 ? c.prof_start() : nullptr;
                    if (e4) fused_ev = e4;
                    cg_fused_launch<T>(c, op.d, Kit, (int)ncol, w, r, p, s, y, st, c1, Gk);
                    if (bs && b == batch - 1) c.prof_stop(fused_ev, 4, n * (es * (ncol + 10.0) + 32.0), iter + 1, batch);
                }
                continue;
            }
            cudaEvent_t e0 = samp ? c.prof_start() : nullptr;
            cg_stencil_dots<T><<<grid_st, 256, 0, c.s>>>(op.d, r, w, st, c.hist.template as<double>(), c.red(), kz);
            c.check_launch();
            if (samp) c.prof_stop(e0, 0, n * (2 * es + 16.0), iter);
            static const int no_tma = [] {
                const char* e = std::getenv("ROMDOT_NO_TMA");
                return e ? std::atoi(e) : 0;
            }();
            if (ncol > 0 && no_tma) {
                ts_T_launch<T, false, true>(c, Kit, ncol, ncol, w, n, c1, st);
                ts_NT_launch<T, false, true>(c, Kit, ncol, ncol, w, w, n, c1, c2, st);
                cg_update<T, true><<<c.grid_for(n, 256, 8), 256, smem_c, c.s>>>(Kit, ncol, (int)ncol, w, n, c2, r, p,
                                                                                s, y, st);
                c.check_launch();
            } else if (ncol > 0 && gram_pass) {
                cudaEvent_t e1 = samp ? c.prof_start() : nullptr;
                ts_tma_launch<T, 0>(c, Kit, (int)ncol, n, w, nullptr, nullptr, c1, nullptr, nullptr, nullptr, nullptr,
                                    st);
                if (samp) c.prof_stop(e1, 1, n * es * (ncol + 1.0), iter);
                cudaEvent_t e3 = samp ? c.prof_start() : nullptr;
                ts_tma_launch<T, 2>(c, Kit, (int)ncol, n, w, nullptr, c1, nullptr, r, p, s, y, st, Gk);
                if (samp) c.prof_stop(e3, 3, n * es * (ncol + 9.0), iter);
            } else if (ncol > 0) {
                static const int tma_mask = [] {
                    const char* e = std::getenv("ROMDOT_TMA_MASK");
                    return e ? std::atoi(e) : 0;
                }();
                cudaEvent_t e1 = samp ? c.prof_start() : nullptr;
                if (tma_mask & 1)
                    ts_T_launch<T, false, true>(c, Kit, ncol, ncol, w, n, c1, st);
                else
                    ts_tma_launch<T, 0>(c, Kit, (int)ncol, n, w, nullptr, nullptr, c1, nullptr, nullptr, nullptr,
                                        nullptr, st);
                if (samp) c.prof_stop(e1, 1, n * es * (ncol + 1.0), iter);
                cudaEvent_t e2 = samp ? c.prof_start() : nullptr;
                if (tma_mask & 2)
                    ts_NT_launch<T, false, true>(c, Kit, ncol, ncol, w, w, n, c1, c2, st);
                else
                    ts_tma_launch<T, 1>(c, Kit, (int)ncol, n, w, w, c1, c2, nullptr, nullptr, nullptr, nullptr, st);
                if (samp) c.prof_stop(e2, 2, n * es * (ncol + 2.0), iter);
                cudaEvent_t e3 = samp ? c.prof_start() : nullptr;
                if (tma_mask & 4) {
                    cg_update<T, true><<<c.grid_for(n, 256, 8), 256, smem_c, c.s>>>(Kit, ncol, (int)ncol, w, n, c2, r,
                                                                                    p, s, y, st);
                    c.check_launch();
                } else {
                    ts_tma_launch<T, 2>(c, Kit, (int)ncol, n, w, nullptr, c2, nullptr, r, p, s, y, st);
                }
                if (samp) c.prof_stop(e3, 3, n * es * (ncol + 9.0), iter);
            } else {
                cudaEvent_t e3 = samp ? c.prof_start() : nullptr;
                cg_update<T, false><<<c.grid_for(n, 256, 8), 256, smem_c, c.s>>>(Kit, n, 0, w, n, c2, r, p, s, y, st);
                c.check_launch();
                if (samp) c.prof_stop(e3, 3, n * es * 9.0, iter);
            }
        }
        ++batches;
    };
    // two batches in flight; poll the done flag of the older one
    int slot = 0;
    launch_batch();
    CK(cudaMemcpyAsync(&c.st_host[0], st, sizeof(CGState), cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.ev[0], c.s));
    launch_batch();
    CK(cudaMemcpyAsync(&c.st_host[1], st, sizeof(CGState), cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.ev[1], c.s));
    long guard = 0;
    while (true) {
        CK(cudaEventSynchronize(c.ev[slot]));
        if (c.st_host[slot].done) break;
        if (++guard > (maxit / batch) + 8) break;
        launch_batch();
        CK(cudaMemcpyAsync(&c.st_host[slot], st, sizeof(CGState), cudaMemcpyDeviceToHost, c.s));
        CK(cudaEventRecord(c.ev[slot], c.s));
        slot ^= 1;
    }
    CK(cudaMemcpyAsync(&c.st_host[0], st, sizeof(CGState), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    const CGState fin = c.st_host[0];
    if (c.prof) c.prof_flush(fin.it);
    c.fprof_report();
    if (c.fchk.p) {  // ROMDOT_FUSED_CHECK: cross-CTA protocol violations of cg_fused
        unsigned bad = 0;
        CK(cudaMemcpy(&bad, c.fchk.p, sizeof(unsigned), cudaMemcpyDeviceToHost));
        c.fchk_violations += bad;
        c.fchk_checked += fused ? std::max(0, fin.it - 1) : 0;
        if (bad) {
            CK(cudaMemset(c.fchk.p, 0, sizeof(unsigned)));
            throw SolverError("cg_fused: " + std::to_string(bad) + " stencil halo reads raced their owner's update");
        }
    }
    SolveOut out;
    out.iterations = fin.it;
    out.converged = fin.converged != 0;
    out.final_relres = fin.relres;
    if (want_hist) {
        const long m = std::min<long>(fin.it + 1, c.hist_cap);
        out.hist.resize(m);
        CK(cudaMemcpy(out.hist.data(), c.hist.p, sizeof(double) * m, cudaMemcpyDeviceToHost));
    }
    CK(cudaMemcpyAsync(y_out, y, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
    y = y_out;
    // image = A y ; g = y + U (e - K^T image)
    launch_stencil<T>(c, op.d, y, n, nullptr, image, n, 1);
    if (ncol > 0) {
        if (padded_io)
            global_T<T, false>(c, K, n, ncol, image, n, c1);
        else
            ts_T_launch<T, false>(c, K, n, ncol, image, n, c1);
        launch_addsub(c, (int)(ncol * W), c1, e, -1.0, c2);  // c2 = K^T image - e
        if (padded_io)
            global_N<T>(c, U, n, ncol, y, g, n, c2);  // g = y - U c2
        else
            ts_N_launch<T>(c, U, n, ncol, y, g, n, c2);
    } else if (g != y) {
        CK(cudaMemcpyAsync(g, y, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
    }
    return out;
}

// The reference's recycled MINRES (krylov.cpp:17-98 minres_core, :147-179
// recycled_minres) on the device, real symmetric operators only: Lanczos on
// (I - K K^T) A started from the projected rhs, every new Lanczos vector
// re-projected against K, Paige-Saunders Givens recurrence for the solution,
// the reference's stopping rules (relres = |phibar| / scale <= tol, NaN
// breakdown, 50-iteration stagnation window, exhausted Krylov space). This is
// the PARITY path (ctx solver = 1, rd_ctx_set_solver): it makes the BuildLog of
// the reference's own solver reproducible on the device. The scalar recurrence
// runs on the host (two small D2H reads per iteration); the product default is
// the device-resident CG above. ncol = 0: plain MINRES (krylov.cpp:100-104).
// g = y + U (K^T rhs - K^T A y) as in recycled_cg (K^T rhs = 0 for every
// right-hand side the builder passes, where this is krylov.cpp:172).
inline SolveOut recycled_minres_dev(Ctx& c, DevOp& op, const double* U, const double* K, long ncol, const double* rhs,
                                    double tol, long maxit, double rhs_scale, double* g, double* y_out, double* image,
                                    Workspace<double>& ws, bool want_hist) {
    const long n = op.n();
    const long npad = padded_rows(n);
    ws.ensure(npad);
    double* v = ws.r.template as<double>();
    double* p = ws.w.template as<double>();
    double* v_old = ws.p.template as<double>();
    double* d_old = ws.s.template as<double>();
    double* d_oold = ws.tmp.template as<double>();
    double* x = ws.y.template as<double>();
    double* e = c.sc(0);
    double* c1 = c.sc(1);
    double* c2 = c.sc(2);
    double* nrm = c.sc(3);
    if (ncol > 1024) throw ConfigError("recycle space wider than 1024 columns");
    const dim3 gv((unsigned)c.grid_for(n, 256, 4));
    auto project = [&](double* wv) {  // w -= K (K^T w) (krylov.cpp:153-155)
        if (ncol == 0) return;
        ts_T_launch<double, false>(c, K, n, ncol, wv, n, c1);
        ts_N_launch<double>(c, K, n, ncol, wv, wv, n, c1);
    };
    auto fetch = [&](const double* d) {
        double h;
        CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        return h;
    };
    auto norm_of = [&](const double* d) {
        launch_norms<double>(c, d, n, nrm);
        return std::sqrt(fetch(nrm));
    };
    if (ncol > 0) ts_T_launch<double, false>(c, K, n, ncol, rhs, n, e);
    CK(cudaMemcpyAsync(v, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.s));
    project(v);  // r0 (krylov.cpp:157-158)
    const double scale = rhs_scale > 0.0 ? rhs_scale : norm_of(rhs);
    const double beta1 = norm_of(v);
    CK(cudaMemsetAsync(x, 0, sizeof(double) * npad, c.s));
    CK(cudaMemsetAsync(v_old, 0, sizeof(double) * npad, c.s));
    CK(cudaMemsetAsync(d_old, 0, sizeof(double) * npad, c.s));
    CK(cudaMemsetAsync(d_oold, 0, sizeof(double) * npad, c.s));
    SolveOut out;
    double relres = 0.0;
    if (beta1 == 0.0 || scale == 0.0) {  // krylov.cpp:26-30
        out.converged = true;
        out.hist.push_back(0.0);
    } else {
        relres = beta1 / scale;
        out.hist.push_back(relres);
        if (relres <= tol) {
            out.converged = true;
        } else {
            vec_div<<<gv, 256, 0, c.s>>>(v, beta1, n);
            c.check_launch();
            double c_old2 = 1.0, s_old2 = 0.0, c_old = 1.0, s_old = 0.0;
            double phibar = beta1, beta = 0.0, best = relres;
            int stagnant = 0;
            for (long k = 1; k <= maxit; ++k) {
                launch_stencil<double>(c, op.d, v, n, nullptr, p, n, 1);
                project(p);  // op = (I - K K^T) A (krylov.cpp:161-165)
                vec_dot<<<gv, 256, 0, c.s>>>(v, p, n, c.red(), nrm);
                c.check_launch();
                const double alpha = fetch(nrm);
                minres_lanczos<<<gv, 256, 0, c.s>>>(p, v, v_old, alpha, beta, n);
                c.check_launch();
                project(p);  // reorth (krylov.cpp:53)
                const double beta_next = norm_of(p);
                const double eps = s_old2 * beta;
                const double delta_bar = c_old2 * beta;
                const double delta = c_old * delta_bar + s_old * alpha;
                const double gamma_bar = -s_old * delta_bar + c_old * alpha;
                const double gamma = std::hypot(gamma_bar, beta_next);
                if (gamma == 0.0) break;  // operator singular on this Krylov space
                const double cs = gamma_bar / gamma;
                const double sn = beta_next / gamma;
                const bool advance = beta_next > 1e-300;
                minres_update<<<gv, 256, 0, c.s>>>(x, v, v_old, p, d_old, d_oold, delta, eps, gamma, cs * phibar,
                                                   advance ? beta_next : 1.0, advance ? 1 : 0, n);
                c.check_launch();
                phibar = -sn * phibar;
                relres = std::abs(phibar) / scale;
                out.iterations = (int)k;
                out.hist.push_back(relres);
                if (!std::isfinite(relres)) break;  // NaN breakdown
                if (relres <= tol) {
                    out.converged = true;
                    break;
                }
                if (relres < best * (1.0 - 1e-12)) {
                    best = relres;
                    stagnant = 0;
                } else if (++stagnant >= 50) {
                    break;
                }
                if (!advance) break;  // Krylov space exhausted
                beta = beta_next;
                c_old2 = c_old;
                s_old2 = s_old;
                c_old = cs;
                s_old = sn;
            }
        }
    }
    out.final_relres = relres;
    if (!want_hist) out.hist.resize(std::min<size_t>(out.hist.size(), 1));  // [0] = init relres for the callers
    CK(cudaMemcpyAsync(y_out, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.s));
    launch_stencil<double>(c, op.d, y_out, n, nullptr, image, n, 1);  // krylov.cpp:170
    if (ncol > 0) {
        ts_T_launch<double, false>(c, K, n, ncol, image, n, c1);
        launch_addsub(c, (int)ncol, c1, e, -1.0, c2);  // c2 = K^T image - e
        ts_N_launch<double>(c, U, n, ncol, y_out, g, n, c2);  // g = y - U c2
    } else if (g != y_out) {
        CK(cudaMemcpyAsync(g, y_out, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.s));
    }
    return out;
}

// Solver selected on the context: 0 CG / COCG (default), 1 the reference's MINRES.
template <class T>
SolveOut recycled_solve(Ctx& c, DevOp& op, const T* U, const T* K, long ncol, const T* rhs, double tol, long maxit,
                        double rhs_scale, T* g, T* y_out, T* image, Workspace<T>& ws, bool want_hist,
                        bool padded_io = false, const T* Gpre = nullptr) {
    if (c.solver == 1) {
        if constexpr (std::is_same<T, double>::value)
            return recycled_minres_dev(c, op, U, K, ncol, rhs, tol, maxit, rhs_scale, g, y_out, image, ws, want_hist);
        else
            throw ConfigError("solver: MINRES (the reference's solver) is real symmetric only; use CG / COCG");
    }
    return recycled_cg<T>(c, op, U, K, ncol, rhs, tol, maxit, rhs_scale, g, y_out, image, ws, want_hist, padded_io, Gpre);
}

// Batched independent CG / COCG on unit right-hand sides b_c = val[c] e_idx[c]
// (the X0 seed solves, basis.cpp:141-149, and the
// full-order transfer, rom.cpp:71-96). X (n x m, ld n) receives the solutions;
// each column runs the single-solve recurrence (cg_recurrence) with its own
// state, scale |val[c]| and the same stopping rules. Two polls in flight.
template <class T>
std::vector<CGState> batched_cg(Ctx& c, DevOp& op, long m, const long* bidx, const double* bval, double tol,
                                long maxit, T* X) {
    constexpr int W = Sc<T>::W;
    constexpr int NV = 2 * W + 1;
    const long n = op.n();
    std::vector<CGState> fin(m);
    if (m <= 0) return fin;
    for (long j = 0; j < m; ++j)
        if (bidx[j] < 0 || bidx[j] >= n) throw ConfigError("batched CG: right-hand side index out of range");
    const size_t bytes = sizeof(T) * n * m;
    DevBuf Rb, Wb, Pb, Sb, stb, cnt, part, ix, vx;
    for (DevBuf* b : {&Rb, &Wb, &Pb, &Sb}) {
        b->ensure(bytes);
        CK(cudaMemsetAsync(b->p, 0, bytes, c.s));
    }
    CK(cudaMemsetAsync(X, 0, bytes, c.s));
    ix.ensure(sizeof(long) * m);
    vx.ensure(sizeof(double) * m);
    CK(cudaMemcpyAsync(ix.p, bidx, sizeof(long) * m, cudaMemcpyHostToDevice, c.s));
    CK(cudaMemcpyAsync(vx.p, bval, sizeof(double) * m, cudaMemcpyHostToDevice, c.s));
    scatter_unit_rhs<T><<<(int)((m + 127) / 128), 128, 0, c.s>>>(Rb.template as<T>(), n, ix.template as<long>(),
                                                                 vx.template as<double>(), (int)m);
    c.check_launch();
    CGState* hs = nullptr;
    CK(cudaMallocHost(&hs, sizeof(CGState) * m * 2));
    struct HostFree {
        CGState* p;
        ~HostFree() { cudaFreeHost(p); }
    } hf{hs};
    for (long j = 0; j < m; ++j) {
        CGState s0{};
        s0.scale = std::fabs(bval[j]);
        s0.tol = tol;
        s0.maxit = (int)std::min<long>(maxit, 0x7fffffff);
        hs[j] = s0;
    }
    stb.ensure(sizeof(CGState) * m);
    CK(cudaMemcpyAsync(stb.p, hs, sizeof(CGState) * m, cudaMemcpyHostToDevice, c.s));
    CK(cudaStreamSynchronize(c.s));
    CGState* st = stb.template as<CGState>();
    cnt.ensure(sizeof(unsigned) * m);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned) * m, c.s));
    const long gxu = std::max(1L, std::min<long>((n + 255) / 256, std::max(8L, 32L * c.sms / m)));
    const dim3 gup((unsigned)gxu, (unsigned)m);
    const int batch = 8;
    // W = A R for all columns through the multi-column TMA stencil (coefficient planes read
    // once per column group instead of once per column), then the per-column merged dots and
    // scalar steps (bd_dots). Columns outside [lo, hi) have finished (polled states).
    const int gxd = (int)std::max(1L, std::min<long>((n + 255) / 256, (long)c.sms));
    part.ensure(sizeof(double) * m * gxd * NV);
    long lo = 0, hi = m;
    auto launch_batch = [&]() {
        if (hi <= lo) return;
        for (int b = 0; b < batch; ++b) {
            launch_stencil<T>(c, op.d, Rb.template as<T>() + (size_t)lo * n, n, nullptr,
                              Wb.template as<T>() + (size_t)lo * n, n, hi - lo);
            bd_dots<T><<<dim3(gxd, (unsigned)(hi - lo)), 256, 0, c.s>>>(
                Rb.template as<T>() + (size_t)lo * n, Wb.template as<T>() + (size_t)lo * n, n, n, st + lo,
                part.template as<double>(), cnt.template as<unsigned>() + lo, nullptr);
            c.check_launch();
            bcg_update<T><<<gup, 256, 0, c.s>>>(Rb.template as<T>(), Pb.template as<T>(), Sb.template as<T>(), X,
                                                Wb.template as<T>(), n, n, st);
            c.check_launch();
        }
    };
    auto shrink = [&](const CGState* h) {
        while (lo < hi && h[lo].done) ++lo;
        while (hi > lo && h[hi - 1].done) --hi;
    };
    auto all_done = [&](const CGState* h) {
        for (long j = 0; j < m; ++j)
            if (!h[j].done) return false;
        return true;
    };
    int slot = 0;
    launch_batch();
    CK(cudaMemcpyAsync(hs, st, sizeof(CGState) * m, cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.ev[0], c.s));
    launch_batch();
    CK(cudaMemcpyAsync(hs + m, st, sizeof(CGState) * m, cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.ev[1], c.s));
    long guard = 0;
    while (true) {
        CK(cudaEventSynchronize(c.ev[slot]));
        if (all_done(hs + slot * m)) break;
        if (++guard > maxit / batch + 8) break;
        shrink(hs + slot * m);
        launch_batch();
        CK(cudaMemcpyAsync(hs + slot * m, st, sizeof(CGState) * m, cudaMemcpyDeviceToHost, c.s));
        CK(cudaEventRecord(c.ev[slot], c.s));
        slot ^= 1;
    }
    CK(cudaMemcpyAsync(hs, st, sizeof(CGState) * m, cudaMemcpyDeviceToHost, c.s));
    c.sync();
    for (long j = 0; j < m; ++j) fin[j] = hs[j];
    return fin;
}

// (C~^T X)[d, s] = val[d] X[idx[d], s] (C~ has one nonzero per column)
template <class T>
__global__ void fom_gather(const T* __restrict__ X, long n, int ns, const long* __restrict__ didx,
                           const double* __restrict__ dval, int nd, T* __restrict__ Psi) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ns * nd) return;
    const int d = e % nd, s = e / nd;
    Psi[e] = Sc<T>::scale(X[(size_t)s * n + didx[d]], dval[d]);
}

// RecycleSpace::from_raw on the device: sequential CGS2 (bilinear for complex)
// of AW's columns; U = W R^-1 formed column by column. W columns are read
// through `wcol` (indices into Wbase) when given.
template <class T>
void from_raw(Ctx& c, long n, long ncol, const T* Wbase, const int* wcol_host, const T* AW, T* U, T* K) {
    constexpr int W = Sc<T>::W;
    double* coef = c.sc(4);
    double* t1 = c.sc(5);
    double* t2 = c.sc(6);
    double* nrm = c.sc(7);
    for (long t = 0; t < ncol; ++t) {
        T* kt = K + (size_t)t * n;
        T* ut = U + (size_t)t * n;
        const T* wsrc = Wbase + (size_t)(wcol_host ? wcol_host[t] : t) * n;
        cgs2<T, false>(c, K, n, t, AW + (size_t)t * n, kt, n, coef, t1, t2);
        launch_norms<T>(c, kt, n, nrm);
        launch_scale<T>(c, kt, kt, n, nrm, 1);
        if (t > 0)
            ts_N_launch<T>(c, U, n, t, wsrc, ut, n, coef);
        else
            CK(cudaMemcpyAsync(ut, wsrc, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        launch_scale<T>(c, ut, ut, n, nrm, 1);
    }
    (void)W;
}


// ------------------------------------------------------------ eigen seed ---
// Small symmetric eigenproblem of the Lanczos tridiagonal (host, m <= a few
// hundred; the reference uses SelfAdjointEigenSolver on T, krylov.cpp:214-221).
static void jacobi_eig(long m, std::vector<double>& T, std::vector<double>& Z) {
    Z.assign((size_t)m * m, 0.0);
    for (long i = 0; i < m; ++i) Z[i + i * m] = 1.0;
    auto at = [&](long i, long j) -> double& { return T[i + j * m]; };
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (long p = 0; p < m; ++p)
            for (long q = 0; q < m; ++q) {
                tot += at(p, q) * at(p, q);
                if (p != q) off += at(p, q) * at(p, q);
            }
        if (off <= 1e-30 * tot || off < 1e-300) break;
        for (long p = 0; p < m; ++p)
            for (long q = p + 1; q < m; ++q) {
                const double apq = at(p, q);
                if (std::fabs(apq) < 1e-300) continue;
                const double th = (at(q, q) - at(p, p)) / (2.0 * apq);
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
                for (long r = 0; r < m; ++r) {
                    const double a = at(r, p), b = at(r, q);
                    at(r, p) = cs * a - sn * b;
                    at(r, q) = sn * a + cs * b;
                }
                for (long r = 0; r < m; ++r) {
                    const double a = at(p, r), b = at(q, r);
                    at(p, r) = cs * a - sn * b;
                    at(q, r) = sn * a + cs * b;
                }
                for (long r = 0; r < m; ++r) {
                    const double a = Z[r + p * m], b = Z[r + q * m];
                    Z[r + p * m] = cs * a - sn * b;
                    Z[r + q * m] = sn * a + cs * b;
                }
            }
    }
}

// smallest_eigenpairs (krylov.cpp:181-280) on the device: shift-invert
// Lanczos on A^-1 with full two-pass reorthogonalisation; A^-1 v by plain CG
// to 1e-12 (no sparse factorisation on the GPU). Ritz check every max(k,10)
// steps against tol * lambda_max (Gershgorin).
static void smallest_eigenpairs_dev(Ctx& c, DevOp& op, long k, double tol, std::vector<double>& lam, double* Uout,
                                    double inner_tol = 1e-10) {
    const long n = op.n();
    if (k < 1 || k > n) throw ConfigError("eigensolver: k out of range");
    if (!(op.lam_max > 0.0)) {
        op_gershgorin<<<c.grid_for(n, 256, 2), 256, 0, c.s>>>(op.d, c.red(), c.sc(3));
        c.check_launch();
        CK(cudaMemcpyAsync(&op.lam_max, c.sc(3), sizeof(double), cudaMemcpyDeviceToHost, c.s));
        c.sync();
    }
    const double lam_max = op.lam_max;
    long mcap = std::min(n, std::max(2 * k + 30, 60L));
    DevBuf Vb, wbuf, ybuf, ibuf, ubuf, aubuf;
    Vb.ensure(sizeof(double) * n * mcap);
    wbuf.ensure(sizeof(double) * n);
    ybuf.ensure(sizeof(double) * n);
    ibuf.ensure(sizeof(double) * n);
    ubuf.ensure(sizeof(double) * n * k);
    aubuf.ensure(sizeof(double) * n);
    Workspace<double> ws;
    double* w = wbuf.template as<double>();
    double* nrm = c.sc(3);
    double* coef = c.sc(4);
    auto V = [&](long j) { return Vb.template as<double>() + (size_t)j * n; };
    auto grow = [&](long want) {
        if (want <= mcap) return;
        const long nc = std::min(n, std::max(want, 2 * mcap));
        DevBuf nb;
        nb.ensure(sizeof(double) * n * nc);
        CK(cudaMemcpyAsync(nb.p, Vb.p, sizeof(double) * n * mcap, cudaMemcpyDeviceToDevice, c.s));
        c.sync();
        std::swap(Vb.p, nb.p);
        std::swap(Vb.bytes, nb.bytes);
        mcap = nc;
    };
    auto host1 = [&](const double* d) {
        double h;
        CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        return h;
    };
    uint64_t seed = 12345;
    auto random_unit = [&](double* v) {
        vec_randn<<<c.grid_for(n, 256, 8), 256, 0, c.s>>>(v, n, seed++);
        c.check_launch();
    };
    random_unit(V(0));
    launch_norms<double>(c, V(0), n, nrm);
    launch_scale<double>(c, V(0), V(0), n, nrm, 0);
    std::vector<double> alphas, betas;
    long m = 0;
    auto ritz = [&]() -> bool {
        if (m < k) return false;
        std::vector<double> T((size_t)m * m, 0.0), Z;
        for (long i = 0; i < m; ++i) {
            T[i + i * m] = alphas[i];
            if (i + 1 < m) T[i + (i + 1) * m] = T[(i + 1) + i * m] = betas[i];
        }
        jacobi_eig(m, T, Z);
        std::vector<long> ord(m);
        for (long i = 0; i < m; ++i) ord[i] = i;
        std::sort(ord.begin(), ord.end(), [&](long a, long b) { return T[a + a * m] > T[b + b * m]; });
        std::vector<double> lm(k);
        double* U = ubuf.template as<double>();
        for (long i = 0; i < k; ++i) {
            // u_i = V_m z_i, normalised
            std::vector<double> z(m);
            for (long t = 0; t < m; ++t) z[t] = -Z[t + ord[i] * m];
            CK(cudaMemcpyAsync(coef, z.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c.s));
            CK(cudaMemsetAsync(ybuf.p, 0, sizeof(double) * n, c.s));
            double* ui = U + (size_t)i * n;
            ts_N_launch<double>(c, V(0), n, m, ybuf.template as<double>(), ui, n, coef);
            launch_norms<double>(c, ui, n, nrm);
            launch_scale<double>(c, ui, ui, n, nrm, 0);
        }
        for (long i = 0; i < k; ++i) {
            double* ui = U + (size_t)i * n;
            double* au = aubuf.template as<double>();
            launch_stencil<double>(c, op.d, ui, n, nullptr, au, n, 1);
            ts_T_launch<double, false>(c, ui, n, 1, au, n, nrm + 16);
            const double li = host1(nrm + 16);
            lm[i] = li;
            // au - li * ui
            vec_axpby<double><<<c.grid_for(n, 256, 8), 256, 0, c.s>>>(n, make_double2(-li, 0.0), ui,
                                                                       make_double2(1.0, 0.0), au);
            c.check_launch();
            launch_norms<double>(c, au, n, nrm);
            const double res = std::sqrt(host1(nrm));
            if (res > tol * lam_max) {
                VLOG(1, "lanczos: ritz pair %ld residual %.3e > %.3e (lambda %.6e)", i, res, tol * lam_max, li);
                return false;
            }
        }
        lam = lm;
        CK(cudaMemcpyAsync(Uout, U, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, c.s));
        c.sync();
        return true;
    };
    const long check_every = std::max(k, 10L);
    while (m < n) {
        grow(m + 1);
        SolveOut so = recycled_cg<double>(c, op, nullptr, nullptr, 0, V(m), inner_tol, std::min(2 * n, 200000L), 0.0, w,
                                          ybuf.template as<double>(), ibuf.template as<double>(), ws, false);
        VLOG(2, "lanczos step %ld: inner CG %d its, relres %.3e, converged %d", m, so.iterations, so.final_relres,
             (int)so.converged);
        ts_T_launch<double, false>(c, V(m), n, 1, w, n, nrm + 16);
        const double alpha = host1(nrm + 16);
        vec_axpby<double><<<c.grid_for(n, 256, 8), 256, 0, c.s>>>(n, make_double2(-alpha, 0.0), V(m),
                                                                   make_double2(1.0, 0.0), w);
        c.check_launch();
        if (m > 0) {
            vec_axpby<double><<<c.grid_for(n, 256, 8), 256, 0, c.s>>>(n, make_double2(-betas[m - 1], 0.0), V(m - 1),
                                                                       make_double2(1.0, 0.0), w);
            c.check_launch();
        }
        // full reorthogonalisation, two passes (CGS2 against V[:, 0..m])
        cgs2<double, false>(c, V(0), n, m + 1, w, w, n, coef, c.sc(5), c.sc(6));
        alphas.push_back(alpha);
        ++m;
        launch_norms<double>(c, w, n, nrm);
        double beta = std::sqrt(host1(nrm));
        if (beta <= 1e-13 * std::fabs(alpha)) {
            if (m >= n) {
                betas.push_back(0.0);
                break;
            }
            random_unit(w);
            cgs2<double, false>(c, V(0), n, m, w, w, n, coef, c.sc(5), c.sc(6));
            launch_norms<double>(c, w, n, nrm);
            launch_scale<double>(c, w, w, n, nrm, 0);
            beta = 0.0;
        } else {
            launch_scale<double>(c, w, w, n, nrm, 0);
        }
        if (m < n) {
            betas.push_back(beta);
            grow(m + 1);
            CK(cudaMemcpyAsync(V(m), w, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.s));
        }
        if (m % check_every == 0 || m == n) {
            const bool ok = ritz();
            VLOG(1, "lanczos: ritz check at m=%ld -> %s", m, ok ? "converged" : "not yet");
            if (ok) return;
        }
        if (m >= 8 * k + 200) throw SolverError("eigensolver: Lanczos did not converge within 8k+200 steps");
    }
    if (ritz()) return;
    throw SolverError("eigensolver: Lanczos did not converge");
}

// ---------------------------------------------------------- global basis ---
constexpr uint8_t kColEigenvector = 0, kColInitialSolution = 1, kColCorrection = 2;
constexpr double kInnerSafety = 0.25;  // basis.cpp:27

// Host callback run by process_system before each RHS (checkpoint-replay
// parity and CPU-baseline sampling): the basis state it sees through
// rd_basis_get / rd_basis_space is the state the reference's loop body
// (basis.cpp:168-205) starts RHS j from. Nonzero return aborts the system.
typedef int (*RhsHook)(void* user, int system_index, long rhs);

// ------------------------------------------- batched deflated solves ---
// BD_M correction solves of one system in flight (bcg_defl.cuh). The caller
// owns the order: load(slot, ...) right after factor_rhs_space left the
// right-hand side's space in gb.Ur / gb.Kr, iterate() a few steps, poll(), then
// finish(slot, ...) forms image = A y and g = y + U (K^T rhs - K^T image) as
// recycled_cg does. ROMDOT_BATCH=0 keeps every solve on the one-solve path.
inline int batch_slots() {  // read per call so a test can compare both paths in one process
    const char* e = std::getenv("ROMDOT_BATCH");
    return e ? std::atoi(e) : 1;
}
inline int batch_width() {  // slots used of BD_M (A/B: ROMDOT_BATCH_SLOTS=8)
    const char* e = std::getenv("ROMDOT_BATCH_SLOTS");
    return std::max(1, std::min(BD_M, e ? std::atoi(e) : BD_M));
}
inline int batch_steps() {
    static const int b = [] {
        const char* e = std::getenv("ROMDOT_BATCH_STEPS");
        return std::max(1, e ? std::atoi(e) : 4);
    }();
    return b;
}

// Bilinear Cholesky of a small Gram on the host: S upper triangular with
// S^T S = G (no conjugation: G = Kt^T Kt of a complex-symmetric recycle block;
// for real data the ordinary Cholesky), Sinv = S^-1, and the 1-norm condition
// estimate of S. m <= 24. Returns false when a pivot is not finite or vanishes.
template <class T> bool chol_bilinear_host(const std::vector<T>& G, long m, std::vector<T>& Sinv, double& kappa1) {
    using Z = std::complex<double>;
    auto toz = [](T v) {
        if constexpr (Sc<T>::W == 1) return Z(v, 0.0);
        else return Z(v.x, v.y);
    };
    auto fromz = [](Z v) {
        if constexpr (Sc<T>::W == 1) return (T)v.real();
        else return make_double2(v.real(), v.imag());
    };
    std::vector<Z> S((size_t)m * m, Z(0.0)), Si((size_t)m * m, Z(0.0));
    double gmax = 0.0;
    for (long j = 0; j < m; ++j) gmax = std::max(gmax, std::abs(toz(G[j + j * m])));
    for (long j = 0; j < m; ++j) {
        for (long i = 0; i <= j; ++i) {
            Z v = toz(G[i + j * m]);
            for (long k = 0; k < i; ++k) v -= S[k + i * m] * S[k + j * m];
            if (i < j) {
                S[i + j * m] = v / S[i + i * m];
            } else {
                if (!std::isfinite(v.real()) || !std::isfinite(v.imag()) || std::abs(v) <= 1e-28 * gmax) return false;
                S[j + j * m] = std::sqrt(v);
            }
        }
    }
    for (long j = 0; j < m; ++j) {  // Si = S^-1 (upper), column by column
        Si[j + j * m] = Z(1.0) / S[j + j * m];
        for (long i = j - 1; i >= 0; --i) {
            Z v(0.0);
            for (long k = i + 1; k <= j; ++k) v += S[i + k * m] * Si[k + j * m];
            Si[i + j * m] = -v / S[i + i * m];
        }
    }
    double n1 = 0.0, n2 = 0.0;
    for (long j = 0; j < m; ++j) {
        double a = 0.0, b = 0.0;
        for (long i = 0; i <= j; ++i) {
            a += std::abs(S[i + j * m]);
            b += std::abs(Si[i + j * m]);
        }
        n1 = std::max(n1, a);
        n2 = std::max(n2, b);
    }
    kappa1 = n1 * n2;
    if (!std::isfinite(kappa1)) return false;
    Sinv.resize((size_t)m * m);
    for (size_t e = 0; e < Sinv.size(); ++e) Sinv[e] = fromz(Si[e]);
    return true;
}

// The two DMMA passes over a 4-row-blocked n x kb block Q (bd_T_eig: C = Q^T X,
// bd_N_eig: X -= Q C) for up to BD_M columns X at once, outside the batched
// iteration: the per-RHS space factorisation projects a right-hand side's
// trailing columns off the system's eigen block with them (one 6+ TB/s stream of
// the block per pass instead of the thin Gram / GEMM kernels' 2-3.5 TB/s).
// Columns are column-major, ld rows apart, and must cover whole row tiles
// (rows % (4 * 32 * 16 / sizeof(T)) == 0) because the tiles come by bulk TMA.
template <class T> struct EigPass {
    static constexpr int M = BD_M;
    Ctx* ctx = nullptr;
    long n = 0, rows = 0, kb = 0;
    BDLayout LT{}, LN{};
    int nstep = 0;
    DevBuf flags;  // CGState[M + 1][M]: row t has done = 0 for the first t entries

    static long row_quantum() { return 4L * 32 * (16 / (long)sizeof(T)); }
    bool usable(long n_, long ku, long cols) const {
        return ku >= 1 && ku <= 64 && cols >= 1 && cols <= M && n_ % row_quantum() == 0;
    }
    template <int NSTEP> void configure_kernels() {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, bd_T_eig<T>));
        CK(cudaFuncSetAttribute(bd_T_eig<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes));
        CK(cudaFuncGetAttributes(&fa, bd_N_eig<T, NSTEP>));
        CK(cudaFuncSetAttribute(bd_N_eig<T, NSTEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes));
        auto stages = [&](int TR, uint32_t xpad) {
            BDLayout L = bd_layout<T>((int)kb, TR, 2, xpad);
            const uint32_t per = L.stride_k + ((L.stride_x * M + 127u) & ~127u);
            const uint32_t fixed = L.total - 2 * per;
            int S = (int)std::min<long>(8, ((long)optin - 2048 - fixed) / per);
            if (S < 2) throw ConfigError("eigen-block passes: shared-memory ring too large");
            return bd_layout<T>((int)kb, TR, S, xpad);
        };
        // T pass: 512-byte segments per column; N pass: twice the rows (8 row groups per
        // 64 complex rows, one per consumer warp)
        const int trT = 32 * (16 / (int)sizeof(T));
        LT = stages(trT, 64);
        LN = stages(2 * trT, 16);
    }
    void configure(Ctx& c, long n_, long rows_, long ku) {
        ctx = &c;
        n = n_;
        rows = rows_;
        kb = ku;
        nstep = kb <= 16 ? 4 : kb <= 32 ? 8 : 16;
        if (nstep == 4) configure_kernels<4>();
        else if (nstep == 8) configure_kernels<8>();
        else configure_kernels<16>();
        if (!flags.p) {
            std::vector<CGState> h((size_t)(M + 1) * M);
            for (int t = 0; t <= M; ++t)
                for (int m = 0; m < M; ++m) h[(size_t)t * M + m].done = m < t ? 0 : 1;
            flags.ensure(sizeof(CGState) * h.size());
            CK(cudaMemcpy(flags.p, h.data(), sizeof(CGState) * h.size(), cudaMemcpyHostToDevice));
        }
    }
    const CGState* first(int t) const { return flags.template as<CGState>() + (size_t)t * M; }
    // out[(m kb + j) W] = sum_rows Q[row, j] X[row, m] for the columns m that st leaves running
    void T_pass(const T* Q4, const T* X, long ld, const CGState* st, double* out) {
        Ctx& c = *ctx;
        const long ntile = rows / LT.TR;
        const int grid = (int)std::max(1L, std::min<long>(ntile, (long)c.sms));
        bd_T_eig<T><<<grid, TMA_THREADS, LT.total, c.s>>>(Q4, n, ntile, LT, X, ld, st, c.red(), out);
        c.check_launch();
    }
    // X[:, m] -= Q coef[m] (coef[(m kb + j) W])
    void N_pass(const T* Q4, T* X, long ld, const CGState* st, const double* coef) {
        Ctx& c = *ctx;
        const long ntile = rows / LN.TR;
        const int grid = (int)std::max(1L, std::min<long>(ntile, (long)c.sms));
        if (nstep == 4)
            bd_N_eig<T, 4><<<grid, TMA_THREADS, LN.total, c.s>>>(Q4, n, ntile, LN, X, ld, st, coef);
        else if (nstep == 8)
            bd_N_eig<T, 8><<<grid, TMA_THREADS, LN.total, c.s>>>(Q4, n, ntile, LN, X, ld, st, coef);
        else
            bd_N_eig<T, 16><<<grid, TMA_THREADS, LN.total, c.s>>>(Q4, n, ntile, LN, X, ld, st, coef);
        c.check_launch();
    }
};

template <class T> struct BatchedDeflated {
    static constexpr int M = BD_M;
    static constexpr int W = Sc<T>::W;
    static constexpr int NV = 2 * W + 1;
    static constexpr int kTS = BD_TCH * BD_NCH;  // slot stride of the trailing coefficient arrays
    Ctx* ctx = nullptr;
    long n = 0, npad = 0, kb = 0, tcap = 0, cmax = 0;
    DevBuf Rb, Wb, Pb, Sb, Yb, Ktb, Utb, Gb, Eb, c1e, c1t, cpe, cpt, stb, krb, part_st, cnt_st, part_tr, cnt_tr, tmp, h0;
    CGState* hs = nullptr;  // pinned: [0, M) polled states, [M, 2M) init staging
    double* h0h = nullptr;  // pinned: relres of iteration 0 per slot (first residual of the solve)
    BDTrail<T> tr{};
    EigPass<T> ep;
    int gx = 1;
    int tw[M] = {0};
    ~BatchedDeflated() {
        if (hs) cudaFreeHost(hs);
        if (h0h) cudaFreeHost(h0h);
        for (auto& e : pev)
            if (e) cudaEventDestroy(e);
    }
    T* col(DevBuf& b, int m) const { return b.template as<T>() + (size_t)m * npad; }
    T* kt(int m) const { return Ktb.template as<T>() + (size_t)m * tcap * npad; }
    T* ut(int m) const { return Utb.template as<T>() + (size_t)m * tcap * npad; }
    double* e_of(int m) const { return Eb.template as<double>() + (size_t)m * cmax * W; }

    static bool supported(long ku, long tmax) { return ku >= 1 && ku <= 64 && tmax <= BD_TCH * BD_NCH; }

    // per system: the eigen block of gb.Kr (n x ku, ld n) in the row-blocked layout
    void begin_system(Ctx& c, const OpDev& op, const T* Kb_colmajor, long ku, long tmax) {
        ctx = &c;
        n = op.n;
        npad = padded_rows(n);
        kb = ku;
        tcap = std::max(1L, tmax);
        cmax = kb + tcap;
        if (!hs) CK(cudaMallocHost(&hs, sizeof(CGState) * 2 * M));
        if (!h0h) CK(cudaMallocHost(&h0h, sizeof(double) * M));
        h0.ensure(sizeof(double) * M);
        CK(cudaMemsetAsync(h0.p, 0, sizeof(double) * M, c.s));
        const size_t vb = sizeof(T) * npad * M;
        for (DevBuf* b : {&Rb, &Wb, &Pb, &Sb, &Yb}) {
            b->ensure(vb);
            CK(cudaMemsetAsync(b->p, 0, vb, c.s));
        }
        tmp.ensure(sizeof(T) * npad * 2);
        CK(cudaMemsetAsync(tmp.p, 0, sizeof(T) * npad * 2, c.s));
        Ktb.ensure(sizeof(T) * npad * tcap * M);
        Utb.ensure(sizeof(T) * npad * tcap * M);
        CK(cudaMemsetAsync(Ktb.p, 0, sizeof(T) * npad * tcap * M, c.s));
        CK(cudaMemsetAsync(Utb.p, 0, sizeof(T) * npad * tcap * M, c.s));
        Gb.ensure(sizeof(T) * cmax * cmax * M);
        Eb.ensure(sizeof(double) * cmax * W * M);
        c1e.ensure(sizeof(double) * kb * W * M);
        cpe.ensure(sizeof(double) * kb * W * M);
        c1t.ensure(sizeof(double) * kTS * W * M);
        cpt.ensure(sizeof(double) * kTS * W * M);
        CK(cudaMemsetAsync(c1t.p, 0, c1t.bytes, c.s));
        stb.ensure(sizeof(CGState) * M);
        for (int m = 0; m < M; ++m) {
            hs[M + m] = CGState{};
            hs[M + m].done = 1;  // empty slot
            tr.Kt[m] = kt(m);
            tr.t[m] = 0;
            tw[m] = 0;
            inuse[m] = false;
        }
        CK(cudaMemcpyAsync(stb.p, hs + M, sizeof(CGState) * M, cudaMemcpyHostToDevice, c.s));
        krb.ensure(sizeof(T) * npad * kb);
        repack_q4<T><<<c.grid_for(npad * kb, 256, 8), 256, 0, c.s>>>(Kb_colmajor, n, (int)kb, n, krb.template as<T>(),
                                                                    npad);
        c.check_launch();
        ep.configure(c, n, npad, kb);
        gx = (int)std::max(1L, std::min<long>((n + 255) / 256, (long)c.sms));
        part_st.ensure(sizeof(double) * M * gx * NV);
        cnt_st.ensure(sizeof(unsigned) * M);
        CK(cudaMemsetAsync(cnt_st.p, 0, sizeof(unsigned) * M, c.s));
        part_tr.ensure(sizeof(double) * M * BD_NCH * gx * BD_TCH * W);
        cnt_tr.ensure(sizeof(unsigned) * M * BD_NCH);
        CK(cudaMemsetAsync(cnt_tr.p, 0, sizeof(unsigned) * M * BD_NCH, c.s));
        c.sync();
    }

    // Slot m takes the solve whose space [Kb | Kt] / [Ub | Ut] (cj = kb + t columns)
    // was factored last into Kr / Ur (ld n) and whose Gram is Gsp (cj x cj).
    // r0 = P rhs by the selective CGS2 of recycled_cg; e = K^T rhs kept for finish().
    void load(int m, const T* Kr, const T* Ur, long cj, const T* Gsp, const T* rhs, double tol, long maxit,
              double scale) {
        Ctx& c = *ctx;
        const long t = cj - kb;
        tw[m] = (int)t;
        tr.t[m] = (int)t;
        if (t > 0) {
            CK(cudaMemcpy2DAsync(kt(m), sizeof(T) * npad, Kr + (size_t)kb * n, sizeof(T) * n, sizeof(T) * n, t,
                                 cudaMemcpyDeviceToDevice, c.s));
            CK(cudaMemcpy2DAsync(ut(m), sizeof(T) * npad, Ur + (size_t)kb * n, sizeof(T) * n, sizeof(T) * n, t,
                                 cudaMemcpyDeviceToDevice, c.s));
        }
        CK(cudaMemcpyAsync(Gb.template as<T>() + (size_t)m * cmax * cmax, Gsp, sizeof(T) * cj * cj,
                           cudaMemcpyDeviceToDevice, c.s));
        launch_norms<T>(c, rhs, n, c.sc(3) + 8);
        c.rflag.ensure(sizeof(CGState));
        cgs2_global_selective<T, false>(c, Kr, n, cj, rhs, col(Rb, m), n, e_of(m), c.sc(1), c.sc(2), c.sc(3) + 8,
                                        c.rflag.template as<CGState>());
        for (DevBuf* b : {&Wb, &Pb, &Sb, &Yb}) CK(cudaMemsetAsync(col(*b, m), 0, sizeof(T) * npad, c.s));
        CGState init{};
        init.scale = scale;
        init.tol = tol;
        init.maxit = (int)std::min<long>(maxit, 0x7fffffff);
        init.hist_cap = 1;  // bd_dots records the first residual (hist0[slot])
        inuse[m] = true;
        last_it[m] = 0;
        hs[M + m] = init;
        CK(cudaMemcpyAsync(stb.template as<CGState>() + m, hs + M + m, sizeof(CGState), cudaMemcpyHostToDevice, c.s));
    }

    void step() {
        Ctx& c = *ctx;
        CGState* st = stb.template as<CGState>();
        const OpDev& op = *opd;
        // stencil over the slots in use (columns 0 .. top; a finished slot inside the range
        // is applied too: its R column is finite and its W column is not read again)
        launch_stencil<T>(c, op, Rb.template as<T>(), npad, nullptr, Wb.template as<T>(), npad, top);
        bd_dots<T><<<dim3(gx, top), 256, 0, c.s>>>(Rb.template as<T>(), Wb.template as<T>(), npad, n, st,
                                                   part_st.template as<double>(), cnt_st.template as<unsigned>(),
                                                   h0.template as<double>());
        c.check_launch();
        ep.T_pass(krb.template as<T>(), Wb.template as<T>(), npad, st, c1e.template as<double>());
        bd_T_trail<T><<<dim3(gx, M), 256, 0, c.s>>>(tr, Wb.template as<T>(), npad, n, st,
                                                    part_tr.template as<double>(), cnt_tr.template as<unsigned>(),
                                                    c1t.template as<double>(), kTS);
        c.check_launch();
        bd_coef<T><<<M, 128, sizeof(T) * cmax, c.s>>>(tr, (int)kb, kTS, st, c1e.template as<double>(),
                                                      c1t.template as<double>(), Gb.template as<T>(), cmax * cmax,
                                                      cpe.template as<double>(), cpt.template as<double>());
        c.check_launch();
        ep.N_pass(krb.template as<T>(), Wb.template as<T>(), npad, st, cpe.template as<double>());
        bd_update<T><<<dim3(gx, M), 256, 0, c.s>>>(tr, Wb.template as<T>(), Rb.template as<T>(), Pb.template as<T>(),
                                                   Sb.template as<T>(), Yb.template as<T>(), npad, n, st,
                                                   cpt.template as<double>(), kTS);
        c.check_launch();
    }
    const OpDev* opd = nullptr;
    int last_it[M] = {0};        // iteration count of each slot at the previous poll
    bool inuse[M] = {false};
    int top = 0;                 // slots [0, top) hold or held a solve in this call
    cudaEvent_t pev[2] = {nullptr, nullptr};
    bool sampled = false;
    void iterate(const OpDev& op, int steps) {
        Ctx& c = *ctx;
        opd = &op;
        top = 0;
        for (int m = 0; m < M; ++m)
            if (inuse[m]) top = m + 1;
        if (top == 0) return;
        sampled = c.prof;
        if (sampled) {
            if (!pev[0])
                for (auto& e : pev) CK(cudaEventCreate(&e));
            CK(cudaEventRecord(pev[0], c.s));
        }
        for (int i = 0; i < steps; ++i) step();
        if (sampled) CK(cudaEventRecord(pev[1], c.s));
    }
    // states of all slots after the queued steps (synchronises the stream).
    // Profile class 5 (rd_ctx_profile): device time of the whole call against
    // the algorithmic bytes of the steps that ran -- per step the eigen block twice
    // (T and N pass) and the 4 coefficient planes once, per slot-step the trailing
    // block twice and 15 vector passes (stencil r, w; T passes w, w; N pass w in and
    // out; update w, r, p, s, y in and r, p, s, y out).
    const CGState* poll() {
        Ctx& c = *ctx;
        CK(cudaMemcpyAsync(hs, stb.p, sizeof(CGState) * M, cudaMemcpyDeviceToHost, c.s));
        CK(cudaMemcpyAsync(h0h, h0.p, sizeof(double) * M, cudaMemcpyDeviceToHost, c.s));
        c.sync();
        if (sampled) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, pev[0], pev[1]));
            const double es = sizeof(T);
            double bytes = 0.0;
            int ran = 0;
            for (int m = 0; m < M; ++m) {
                const int d = std::max(0, hs[m].it - last_it[m]);
                ran = std::max(ran, d);
                bytes += (double)d * es * n * (2.0 * tw[m] + 15.0);
            }
            bytes += (double)ran * n * (2.0 * es * kb + 32.0);
            c.pc[5].ms += ms;
            c.pc[5].bytes += bytes;
            c.pc[5].samples += ran;
            for (int m = 0; m < M; ++m) c.pc[6].samples += std::max(0, hs[m].it - last_it[m]);  // slot-steps
            c.pc[6].ms += ms;
            sampled = false;
        }
        for (int m = 0; m < M; ++m) last_it[m] = hs[m].it;
        return hs;
    }
    // y (padded column of the slot), image = A y (padded), g = y + U (e - K^T image)
    void finish(int m, DevOp& op, const T* Kb_cm, const T* Ub_cm, T* g, T* y_out, T* image) {
        Ctx& c = *ctx;
        const long t = tw[m];
        const long cj = kb + t;
        const T* y = col(Yb, m);
        double* c1 = c.sc(1);
        double* c2 = c.sc(2);
        launch_stencil<T>(c, op.d, y, n, nullptr, image, n, 1);
        global_T<T, false>(c, Kb_cm, n, kb, image, n, c1);
        if (t > 0) global_T<T, false>(c, kt(m), npad, t, image, n, c1 + kb * W);
        launch_addsub(c, (int)(cj * W), c1, e_of(m), -1.0, c2);  // c2 = K^T image - e
        if (t > 0) {
            T* g1 = tmp.template as<T>();
            global_N<T>(c, Ub_cm, n, kb, y, g1, n, c2);
            global_N<T>(c, ut(m), npad, t, g1, g, n, c2 + kb * W);
        } else {
            global_N<T>(c, Ub_cm, n, kb, y, g, n, c2);
        }
        if (y_out) CK(cudaMemcpyAsync(y_out, y, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        // the slot is empty again
        inuse[m] = false;
        last_it[m] = 0;
        hs[M + m] = CGState{};
        hs[M + m].done = 1;
        tr.t[m] = 0;
        tw[m] = 0;
    }
    void release(int m) {
        Ctx& c = *ctx;
        CK(cudaMemcpyAsync(stb.template as<CGState>() + m, hs + M + m, sizeof(CGState), cudaMemcpyHostToDevice, c.s));
    }
};

struct BasisBase {
    virtual ~BasisBase() = default;
    RhsHook hook = nullptr;
    void* hook_user = nullptr;
};

template <class T> struct DevBasis : BasisBase {
    Ctx* ctx = nullptr;
    long n = 0;
    long cols = 0, capcols = 0, ku = 0, cap = 0;
    DevBuf V, Wm, K;            // n x capcols each; W = V R^-1, K = K_img
    std::vector<T> R;           // host, cols x cols column-major (ld = capcols)
    std::vector<uint8_t> markers;
    std::vector<std::vector<int>> spaces;
    bool factored = false;
    bool raw_only = false;  // per-RHS-only comparator: V and the index lists only (no image factor)
    Workspace<T> ws;
    DevBuf tmpv, tmpv2, AW, Ur, Kr, idx, X, bvec;
    DevBuf Ktmp, Gd, Sinvd, Rd, Rd2, gwork;   // block refresh workspace
    DevBuf G00, Gt, Gsp;                     // bilinear Gram of the eigen block / of the current space
    // process_system temporaries, persistent across systems (a multi-GB
    // free + malloc per system costs a device sync and up to ~1 s)
    DevBuf ps_idx, ps_val, ps_Wc, ps_Rall, ps_Coef, ps_Cpk, ps_rj, ps_wn, ps_y, ps_g, ps_im, ps_nrm;
    std::unique_ptr<BatchedDeflated<T>> bd;  // batched solves of the independent right-hand sides
    EigPass<T> ep;                            // DMMA passes over the system's eigen block (space factorisation)
    DevBuf Kq4, Uq4, Gtt, Cee;                // 4-row-blocked copies of Kr / Ur's leading ku columns; Gram pieces
    bool ep_ready = false;
    long stats_batched_rhs = 0, stats_rhs_cgs_fallback = 0;
    // grow-only with 25% slack
    static void grow_to(DevBuf& b, size_t bytes) {
        if (bytes > b.bytes) b.ensure(bytes + bytes / 4);
    }
    long eig_ready_for = -1;                 // system tag whose eig-block factor sits in Ur/Kr
    long cmax_space = 0;
    long stats_block_refresh = 0, stats_seq_refresh = 0, stats_second_pass = 0, stats_rhs_second_pass = 0;

    T* Vp() const { return V.template as<T>(); }
    T* Wp() const { return Wm.template as<T>(); }
    T* Kp() const { return K.template as<T>(); }

    void reserve(long want) {
        if (want <= capcols) return;
        long nc = std::max(want, std::max(16L, capcols * 3 / 2));
        if (cap > 0) nc = std::max(want, cap);  // capped bases are allocated once
        auto grow = [&](DevBuf& b) {
            DevBuf nb;
            nb.ensure(sizeof(T) * n * nc);
            if (b.p && cols > 0) CK(cudaMemcpyAsync(nb.p, b.p, sizeof(T) * n * cols, cudaMemcpyDeviceToDevice, ctx->s));
            ctx->sync();
            std::swap(b.p, nb.p);
            std::swap(b.bytes, nb.bytes);
        };
        grow(V);
        if (!raw_only) {
            grow(Wm);
            grow(K);
        }
        std::vector<T> R2((size_t)nc * nc, Sc<T>::zero());
        for (long j = 0; j < cols; ++j)
            for (long i = 0; i <= j; ++i) R2[i + j * nc] = R[i + j * capcols];
        R.swap(R2);
        capcols = nc;
    }
    T& Rat(long i, long j) { return R[i + j * capcols]; }

    // W = V R^-1 is only read by the refresh and the deferred X assembly, so the
    // appends of a system leave their W columns unformed (one N pass over W per
    // append saved) and materialize_W() forms them as a block:
    //   W_new = (V_new - W_old R_on) R_nn^-1
    // (one tall GEMM over W_old, then forward substitution inside the new block).
    // wvalid = leading columns of W that are formed. ROMDOT_LAZY_W=0 forms each
    // column at its append as before.
    long wvalid = 0;
    DevBuf wblk, wrho;
    static bool lazy_w() {
        static const bool on = [] {
            const char* e = std::getenv("ROMDOT_LAZY_W");
            return e ? std::atoi(e) != 0 : true;
        }();
        return on;
    }
    void materialize_W() {
        if (raw_only || wvalid >= cols) return;
        Ctx& c = *ctx;
        constexpr int W = Sc<T>::W;
        const long m0 = wvalid, m = cols - m0;
        T* Wn = Wp() + (size_t)m0 * n;
        CK(cudaMemcpy2DAsync(Wn, sizeof(T) * n, Vp() + (size_t)m0 * n, sizeof(T) * n, sizeof(T) * n, m,
                             cudaMemcpyDeviceToDevice, c.s));
        // R_on (m0 x m, ld m0) and R_nn (m x m, ld m) to the device, 1 / R_jj^2 as rho^2
        std::vector<T> h((size_t)m0 * m + (size_t)m * m, Sc<T>::zero());
        std::vector<double> r2(m);
        for (long j = 0; j < m; ++j) {
            for (long i = 0; i < m0; ++i) h[i + j * m0] = Rat(i, m0 + j);
            for (long i = 0; i < j; ++i) h[(size_t)m0 * m + i + j * m] = Rat(m0 + i, m0 + j);
            r2[j] = Sc<T>::abs2(Rat(m0 + j, m0 + j));
        }
        wblk.ensure(sizeof(T) * h.size());
        wrho.ensure(sizeof(double) * m);
        CK(cudaMemcpyAsync(wblk.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c.s));
        CK(cudaMemcpyAsync(wrho.p, r2.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c.s));
        const T* Ron = wblk.template as<T>();
        const T* Rnn = Ron + (size_t)m0 * m;
        if (m0 > 0) gemm<T, true>(c, Wp(), n, m0, Ron, m, Wn, n, Wn, n, n, false);
        T* vp = padded(vpad);
        for (long j = 0; j < m; ++j) {
            T* wj = Wn + (size_t)j * n;
            if (j > 0) {
                CK(cudaMemcpyAsync(vp, wj, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
                global_N<T>(c, Wn, n, j, vp, vp, n, (const double*)(Rnn + (size_t)j * m));
                launch_scale<T>(c, vp, wj, n, wrho.template as<double>() + j, 0);
            } else {
                launch_scale<T>(c, wj, wj, n, wrho.template as<double>(), 0);
            }
        }
        c.sync();  // host copies above are stack-owned
        wvalid = cols;
        (void)W;
    }

    void drop_column(long cidx) {
        // V columns shift left; per-RHS indices remapped (SURVEY §5 latent bug fixed)
        for (long k = cidx; k + 1 < cols; ++k)
            CK(cudaMemcpyAsync(Vp() + k * n, Vp() + (k + 1) * n, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->s));
        markers.erase(markers.begin() + cidx);
        for (auto& sp : spaces) {
            std::vector<int> o;
            for (int v : sp) {
                if (v == cidx) continue;
                o.push_back(v > cidx ? v - 1 : v);
            }
            sp.swap(o);
        }
        --cols;
    }

    // Factor column j of V against K[:, :j] at the operator's current fields:
    // z = A_i v_j, CGS2 (Hermitian), K_j = q/rho, W_j = (v_j - W c)/rho, R(:, j).
    // Returns rho / ||z|| decision data; writes nothing if dropped.
    bool factor_column(DevOp& op, long j, bool may_drop) {
        Ctx& c = *ctx;
        constexpr int W = Sc<T>::W;
        tmpv.ensure(sizeof(T) * n);
        T* z = tmpv.template as<T>();
        T* vj = Vp() + (size_t)j * n;
        launch_stencil<T>(c, op.d, vj, n, nullptr, z, n, 1);
        return factor_image(j, vj, z, may_drop);
        (void)W;
    }

    // Padded (zero-tailed) device vectors for the TMA passes over the basis.
    DevBuf zpad, qpad, vpad;
    T* padded(DevBuf& b) {
        if (b.bytes < sizeof(T) * padded_rows(n)) {
            b.ensure(sizeof(T) * padded_rows(n));
            CK(cudaMemsetAsync(b.p, 0, b.bytes, ctx->s));
        }
        return b.template as<T>();
    }

    bool factor_image(long j, const T* vj, const T* z, bool may_drop) {
        Ctx& c = *ctx;
        constexpr int W = Sc<T>::W;
        T* zp = padded(zpad);
        T* qp = padded(qpad);
        T* vp = padded(vpad);
        if (zp != z) CK(cudaMemcpyAsync(zp, z, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
        double* coef = c.sc(4);
        double* nrm = c.sc(7);
        launch_norms<T>(c, zp, n, nrm + 8);
        c.rflag.ensure(sizeof(CGState));
        cgs2_global_selective<T, true>(c, Kp(), n, j, zp, qp, n, coef, c.sc(5), c.sc(6), nrm + 8,
                                       c.rflag.template as<CGState>());
        launch_norms<T>(c, qp, n, nrm);
        std::vector<double> hc(2 + (size_t)j * W);
        CK(cudaMemcpyAsync(hc.data(), nrm, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        CK(cudaMemcpyAsync(hc.data() + 1, nrm + 8, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        if (j > 0) CK(cudaMemcpyAsync(hc.data() + 2, coef, sizeof(double) * j * W, cudaMemcpyDeviceToHost, c.s));
        c.sync();
        const double rho = std::sqrt(hc[0]);
        const double zn = std::sqrt(hc[1]);
        if (may_drop && rho <= 1e-12 * zn) return false;
        launch_scale<T>(c, qp, Kp() + (size_t)j * n, n, nrm, 0);  // K_img(:, j) = q / rho
        T* wj = Wp() + (size_t)j * n;
        if (lazy_w()) {
            // W(:, j) formed later by materialize_W (needs W(:, :j) formed only then)
        } else if (j > 0) {  // W(:, :j) formed: wvalid == j on this path
            CK(cudaMemcpyAsync(vp, vj, sizeof(T) * n, cudaMemcpyDeviceToDevice, c.s));
            global_N<T>(c, Wp(), n, j, vp, vp, n, coef);             // W(:, j) = (v_j - W c) / rho
            launch_scale<T>(c, vp, wj, n, nrm, 0);
            wvalid = j + 1;
        } else {
            launch_scale<T>(c, vj, wj, n, nrm, 0);
            wvalid = 1;
        }
        for (long i = 0; i < j; ++i) {
            if constexpr (W == 1)
                Rat(i, j) = hc[2 + i];
            else
                Rat(i, j) = make_double2(hc[2 + 2 * i], hc[3 + 2 * i]);
        }
        Rat(j, j) = Sc<T>::from(rho);
        return true;
    }

    // GlobalBasis::refresh (basis.cpp:37-76): K_img R = A_i V with drop rule
    // |R_ii| <= 1e-12 ||A_i v_i|| for i >= ku.
    // First call: sequential CGS2 factorisation of every column. Later calls
    // reuse W = V R^-1 of the previous system: Y = A_i W is close to
    // orthonormal (A_i A_{i-1}^-1 ~ I), so one Gram + Cholesky (CholQR) gives
    // K_img = Y S^-1, W <- W S^-1, R <- S R; a second pass only if kappa(S)
    // is large. Any pivot failure or deficient column falls back to the
    // sequential path (which drops columns like the reference).
    void refresh(DevOp& op) {
        eig_ready_for = -1;
        if (factored && cols > 0) {
            materialize_W();
            if (refresh_block(op)) {
                ++stats_block_refresh;
                return;
            }
        }
        ++stats_seq_refresh;
        wvalid = 0;  // every column is refactored: W is formed again from V
        long j = 0;
        while (j < cols) {
            if (factor_column(op, j, j >= ku)) {
                ++j;
            } else {
                drop_column(j);
            }
        }
        factored = true;
        materialize_W();
    }

    bool refresh_block(DevOp& op) {
        Ctx& c = *ctx;
        const long r = cols;
        Ktmp.ensure(sizeof(T) * n * capcols);
        Gd.ensure(sizeof(T) * r * r);
        Sinvd.ensure(sizeof(T) * r * r);
        Rd.ensure(sizeof(T) * r * r);
        Rd2.ensure(sizeof(T) * r * r);
        launch_stencil<T>(c, op.d, Wp(), n, nullptr, Ktmp.template as<T>(), n, r);  // Y = A_i W
        // upload R (ld r)
        std::vector<T> Rh((size_t)r * r, Sc<T>::zero());
        for (long j = 0; j < r; ++j)
            for (long i = 0; i <= j; ++i) Rh[i + j * r] = Rat(i, j);
        CK(cudaMemcpyAsync(Rd.p, Rh.data(), sizeof(T) * r * r, cudaMemcpyHostToDevice, c.s));
        for (int pass = 0; pass < 2; ++pass) {
            // pass 0 factors Y (in Ktmp); pass 1 re-orthogonalises K_img
            const T* src = pass == 0 ? Ktmp.template as<T>() : Kp();
            gram<T, true>(c, src, n, r, src, n, r, n, Gd.template as<T>(), true, gwork);
            CholInfo ci = chol_inv<T, true>(c, Gd.template as<T>(), Sinvd.template as<T>(), r, true);
            if (ci.bad) return false;
            if (pass == 0) {
                gemm<T, false>(c, src, n, r, Sinvd.template as<T>(), r, nullptr, 0, Kp(), n, n, true);
            } else {
                gemm<T, false>(c, src, n, r, Sinvd.template as<T>(), r, nullptr, 0, Ktmp.template as<T>(), n, n, true);
                std::swap(K.p, Ktmp.p);
                std::swap(K.bytes, Ktmp.bytes);
            }
            gemm<T, false>(c, Wp(), n, r, Sinvd.template as<T>(), r, nullptr, 0, Ktmp.template as<T>(), n, n, true);
            std::swap(Wm.p, Ktmp.p);
            std::swap(Wm.bytes, Ktmp.bytes);
            tri_mul_upper<T><<<c.grid_for(r * r, 256, 4), 256, 0, c.s>>>(Gd.template as<T>(), Rd.template as<T>(),
                                                                           Rd2.template as<T>(), (int)r, (int)r);
            c.check_launch();
            std::swap(Rd.p, Rd2.p);
            std::swap(Rd.bytes, Rd2.bytes);
            VLOG(1, "refresh pass %d: r %ld, kappa1(S) %.3e", pass, r, ci.kappa1);
            if (ci.kappa1 <= refresh_kappa()) break;
            ++stats_second_pass;
        }
        CK(cudaMemcpyAsync(Rh.data(), Rd.p, sizeof(T) * r * r, cudaMemcpyDeviceToHost, c.s));
        c.sync();
        // deficiency check (basis.cpp:57-61): |R_ii| <= 1e-12 ||R(:, i)|| = 1e-12 ||A_i v_i||
        for (long i = ku; i < r; ++i) {
            double cn = 0.0;
            for (long k = 0; k <= i; ++k) cn += Sc<T>::abs2(Rh[k + i * r]);
            if (std::sqrt(Sc<T>::abs2(Rh[i + i * r])) <= 1e-12 * std::sqrt(cn)) {
                factored = false;  // sequential path re-factors and drops
                return false;
            }
        }
        for (long j = 0; j < r; ++j)
            for (long i = 0; i <= j; ++i) Rat(i, j) = Rh[i + j * r];
        return true;
    }

    // ---- per-RHS recycle spaces (RecycleSpace::from_raw, krylov.cpp:106-115) ----
    // U_j = V[:, idx_j] with idx_j = [0..ku) + trailing columns. The eigen block
    // [0..ku) is shared by every RHS of a system, so its factor A_i U0 = Q0 S0
    // (bilinear for complex) and P0 = U0 S0^-1 are computed once per system
    // into the leading columns of Kr / Ur; per RHS only the trailing columns
    // are projected against Q0 (block CGS2) and orthonormalised (CGS2).
    // Same span and projector as the reference's full per-RHS QR.
    void factor_eig_block(DevOp& op, long cspace) {
        Ctx& c = *ctx;
        // the widest space grows by about one column per system: allocate with
        // 16 columns of slack so these multi-GB buffers are not re-allocated
        // (device sync + free + malloc) every system
        const long cs = std::max(1L, cspace) + 16;
        if ((size_t)(sizeof(T) * n * std::max(1L, cspace)) > Ur.bytes) Ur.ensure(sizeof(T) * n * cs);
        if ((size_t)(sizeof(T) * n * std::max(1L, cspace)) > Kr.bytes) Kr.ensure(sizeof(T) * n * cs);
        if ((size_t)(sizeof(T) * n * std::max(ku, cspace)) > AW.bytes) AW.ensure(sizeof(T) * n * std::max(ku, cs));
        tmpv2.ensure(sizeof(T) * n);
        if (ku == 0) return;
        T* Kb = Kr.template as<T>();
        T* Ub = Ur.template as<T>();
        T* S = AW.template as<T>();
        Gd.ensure(sizeof(T) * ku * ku);
        Sinvd.ensure(sizeof(T) * ku * ku);
        launch_stencil<T>(c, op.d, Vp(), n, nullptr, Kb, n, ku);  // A_i U0
        CK(cudaMemcpyAsync(Ub, Vp(), sizeof(T) * n * ku, cudaMemcpyDeviceToDevice, c.s));
        for (int pass = 0; pass < 3; ++pass) {
            gram<T, false>(c, Kb, n, ku, Kb, n, ku, n, Gd.template as<T>(), true, gwork);
            CholInfo ci = chol_inv<T, false>(c, Gd.template as<T>(), Sinvd.template as<T>(), ku, true);
            if (ci.bad) throw SolverError("recycle space: eigen block image is numerically singular");
            gemm<T, false>(c, Kb, n, ku, Sinvd.template as<T>(), ku, nullptr, 0, S, n, n, true);
            CK(cudaMemcpyAsync(Kb, S, sizeof(T) * n * ku, cudaMemcpyDeviceToDevice, c.s));
            gemm<T, false>(c, Ub, n, ku, Sinvd.template as<T>(), ku, nullptr, 0, S, n, n, true);
            CK(cudaMemcpyAsync(Ub, S, sizeof(T) * n * ku, cudaMemcpyDeviceToDevice, c.s));
            if (ci.kappa1 <= 20.0) break;
        }
        // G00 = Q0^T Q0 of the final eigen-block factor (shared by every RHS's
        // space Gram, used by the one-pass inner projection)
        G00.ensure(sizeof(T) * ku * ku);
        gram<T, false>(c, Kb, n, ku, Kb, n, ku, n, G00.template as<T>(), true, gwork);
        // 4-row-blocked copies for the DMMA passes of factor_rhs_space / space_gram
        static const int use_ep = [] {
            const char* e = std::getenv("ROMDOT_RHS_DMMA");
            return e ? std::atoi(e) : 1;
        }();
        ep_ready = use_ep && ep.usable(n, ku, 1);
        if (ep_ready) {
            ep.configure(c, n, n, ku);
            Kq4.ensure(sizeof(T) * n * ku);
            Uq4.ensure(sizeof(T) * n * ku);
            repack_q4<T><<<c.grid_for(n * ku, 256, 8), 256, 0, c.s>>>(Kb, n, (int)ku, n, Kq4.template as<T>(), n);
            c.check_launch();
            repack_q4<T><<<c.grid_for(n * ku, 256, 8), 256, 0, c.s>>>(Ub, n, (int)ku, n, Uq4.template as<T>(), n);
            c.check_launch();
        }
    }

    // G = K^T K of the space factored last (ku + m columns): G00 plus the thin
    // block [Q0 Kt]^T Kt in <= 8-column chunks. Returns the device pointer.
    const T* space_gram(long cj) {
        Ctx& c = *ctx;
        const long m = cj - ku;
        Gsp.ensure(sizeof(T) * std::max(1L, cj * cj));
        if (m <= 0) return ku > 0 ? G00.template as<T>() : nullptr;
        T* Kb = Kr.template as<T>();
        const T* Kt = Kb + (size_t)ku * n;
        Gt.ensure(sizeof(T) * cj * m);
        if (ep_ready && ep.usable(n, ku, m)) {
            // [Kb Kt]^T Kt in two pieces: Kb^T Kt by the DMMA T pass (one stream of the eigen
            // block), Kt^T Kt by the thin Gram over the trailing columns only
            Cee.ensure(sizeof(double) * Sc<T>::W * ku * BD_M);
            Gtt.ensure(sizeof(T) * m * m);
            ep.T_pass(Kq4.template as<T>(), Kt, n, ep.first((int)m), Cee.template as<double>());
            for (long t0 = 0; t0 < m; t0 += 8) {
                const long b = std::min(8L, m - t0);
                gram<T, false>(c, Kt, n, m, Kt + (size_t)t0 * n, n, b, n, Gtt.template as<T>() + (size_t)t0 * m, false,
                               gwork);
            }
            stack_space_gt<T><<<c.grid_for(cj * m, 256, 1), 256, 0, c.s>>>(Cee.template as<T>(), (int)ku,
                                                                            Gtt.template as<T>(), (int)m,
                                                                            Gt.template as<T>());
            c.check_launch();
        } else {
            for (long t0 = 0; t0 < m; t0 += 8) {
                const long b = std::min(8L, m - t0);
                gram<T, false>(c, Kb, n, cj, Kt + (size_t)t0 * n, n, b, n, Gt.template as<T>() + (size_t)t0 * cj,
                               false, gwork);
            }
        }
        assemble_space_gram<T><<<c.grid_for(cj * cj, 256, 1), 256, 0, c.s>>>(
            ku > 0 ? G00.template as<T>() : nullptr, (int)ku, Gt.template as<T>(), (int)cj, Gsp.template as<T>());
        c.check_launch();
        return Gsp.template as<T>();
    }

    void factor_rhs_space(DevOp& op, const std::vector<int>& cidx) {
        Ctx& c = *ctx;
        constexpr int W = Sc<T>::W;
        const long cj = (long)cidx.size();
        const long m = cj - ku;
        T* Kb = Kr.template as<T>();
        T* Ub = Ur.template as<T>();
        if (m <= 0) return;
        T* Kt = Kb + (size_t)ku * n;
        T* Ut = Ub + (size_t)ku * n;
        idx.ensure(sizeof(int) * m);
        CK(cudaMemcpyAsync(idx.p, cidx.data() + ku, sizeof(int) * m, cudaMemcpyHostToDevice, c.s));
        launch_stencil<T>(c, op.d, Vp(), n, idx.template as<int>(), Kt, n, m);
        for (long t = 0; t < m; ++t)
            CK(cudaMemcpyAsync(Ut + (size_t)t * n, Vp() + (size_t)cidx[ku + t] * n, sizeof(T) * n,
                               cudaMemcpyDeviceToDevice, c.s));
        dbg_sum(" frs stencil", Kt, n * m, c.s);
        if (ku > 0) {
            T* C1 = (T*)c.sc(4);
            T* C2 = (T*)c.sc(5);
            if (ku * m * W > 8192) throw ConfigError("recycle space: trailing block too wide");
            static const int onepass = [] {
                // default on: C4 per-RHS spaces 420 -> 300 ms per late system; GPU suite and
                // the C4 partial lockstep (profiles/r01g_rhs_onepass.txt) unchanged
                const char* e = std::getenv("ROMDOT_RHS_ONEPASS");
                return e ? std::atoi(e) : 1;
            }();
            if (onepass) {
                // one T and one N pass over the eigen block (Gram-corrected coefficient,
                // G00 = Kb^T Kb formed with the eigen block) instead of two each.
                // The Gram correction equals CGS2 only in exact arithmetic, so the
                // Kahan-Parlett guard of the global appends applies: when a column
                // lost more than half of ||kt||^2 to the projection (cancellation),
                // a second plain pass (C = Kb^T Kt ; Kt -= Kb C ; Ut -= Ub C) repairs
                // the loss of orthogonality. The column norms are one extra read of
                // the m trailing columns each side of the projection.
                double* nb = c.sc(10);
                double* na = c.sc(11);
                col_norms<T><<<c.grid_for(n, 256, 2), 256, sizeof(double) * m, c.s>>>(Kt, n, (int)m, n, c.red(), nb);
                c.check_launch();
                // the three passes over the eigen block: bd_T_eig / bd_N_eig (DMMA, one bulk-TMA
                // stream of the 4-row-blocked block per pass) when the shape allows, else the
                // thin Gram / GEMM kernels
                const bool dm = ep_ready && ep.usable(n, ku, m);
                auto T_pass = [&](T* Cout) {
                    if (dm)
                        ep.T_pass(Kq4.template as<T>(), Kt, n, ep.first((int)m), (double*)Cout);
                    else
                        gram<T, false>(c, Kb, n, ku, Kt, n, m, n, Cout, false, gwork);
                };
                auto N_pass = [&](const T* Cin) {
                    if (dm) {
                        ep.N_pass(Kq4.template as<T>(), Kt, n, ep.first((int)m), (const double*)Cin);
                        ep.N_pass(Uq4.template as<T>(), Ut, n, ep.first((int)m), (const double*)Cin);
                    } else {
                        gemm<T, true>(c, Kb, n, ku, Cin, m, Kt, n, Kt, n, n, false);
                        gemm<T, true>(c, Ub, n, ku, Cin, m, Ut, n, Ut, n, n, false);
                    }
                };
                T_pass(C1);
                onepass_coef<T><<<c.grid_for(ku * m, 256, 1), 256, 0, c.s>>>(G00.template as<T>(), (int)ku, C1,
                                                                               (int)m, C2);
                c.check_launch();
                N_pass(C2);
                col_norms<T><<<c.grid_for(n, 256, 2), 256, sizeof(double) * m, c.s>>>(Kt, n, (int)m, n, c.red(), na);
                c.check_launch();
                std::vector<double> hn(2 * m);
                CK(cudaMemcpyAsync(hn.data(), nb, sizeof(double) * m, cudaMemcpyDeviceToHost, c.s));
                CK(cudaMemcpyAsync(hn.data() + m, na, sizeof(double) * m, cudaMemcpyDeviceToHost, c.s));
                c.sync();
                bool cancel = false;
                for (long t = 0; t < m; ++t) cancel |= hn[m + t] < 0.5 * hn[t];
                if (cancel) {
                    ++stats_rhs_second_pass;
                    T_pass(C1);
                    N_pass(C1);
                }
            } else {
                gram<T, false>(c, Kb, n, ku, Kt, n, m, n, C1, false, gwork);
                dbg_sum(" frs C1", C1, ku * m, c.s);
                gemm<T, true>(c, Kb, n, ku, C1, m, Kt, n, Kt, n, n, false);
                dbg_sum(" frs Kt1", Kt, n * m, c.s);
                gram<T, false>(c, Kb, n, ku, Kt, n, m, n, C2, false, gwork);
                dbg_sum(" frs C2", C2, ku * m, c.s);
                gemm<T, true>(c, Kb, n, ku, C2, m, Kt, n, Kt, n, n, false);
                dbg_sum(" frs Kt2", Kt, n * m, c.s);
                launch_addsub(c, (int)(ku * m * W), (double*)C1, (double*)C2, 1.0, (double*)C1);
                gemm<T, true>(c, Ub, n, ku, C1, m, Ut, n, Ut, n, n, false);
                dbg_sum(" frs Ut", Ut, n * m, c.s);
            }
        }
        // Trailing block: bilinear CholQR. G = Kt^T Kt (thin Gram over the m trailing columns),
        // S^T S = G factored on the host (m <= 24), Kt <- Kt S^-1 and Ut <- Ut S^-1 in place;
        // repeated while the factor's condition estimate says the pass lost digits (the rule of
        // the eigen block above). A dozen launches instead of nine per column; same span and
        // triangular structure as the column-by-column CGS2 below, which stays the fallback
        // when the factor breaks down (ROMDOT_RHS_CHOLQR=0: always CGS2).
        static const int cholqr = [] {
            const char* e = std::getenv("ROMDOT_RHS_CHOLQR");
            return e ? std::atoi(e) : 1;
        }();
        if (cholqr && m >= 2 && m <= 24) {
            bool ok = true;
            Gtt.ensure(sizeof(T) * 2 * m * m);
            T* Gd_ = Gtt.template as<T>();
            T* Sd_ = Gd_ + (size_t)m * m;
            std::vector<T> hG((size_t)m * m), hS;
            for (int pass = 0; pass < 3 && ok; ++pass) {
                for (long t0 = 0; t0 < m; t0 += 8) {
                    const long b = std::min(8L, m - t0);
                    gram<T, false>(c, Kt, n, m, Kt + (size_t)t0 * n, n, b, n, Gd_ + (size_t)t0 * m, false, gwork);
                }
                CK(cudaMemcpyAsync(hG.data(), Gd_, sizeof(T) * m * m, cudaMemcpyDeviceToHost, c.s));
                c.sync();
                double kappa = 0.0;
                if (!chol_bilinear_host<T>(hG, m, hS, kappa)) {
                    ok = false;
                    break;
                }
                CK(cudaMemcpyAsync(Sd_, hS.data(), sizeof(T) * m * m, cudaMemcpyHostToDevice, c.s));
                const int grid = c.grid_for(n, 256, 8);
                auto apply = [&](T* X) {
                    if (m <= 4) tri_right_inplace<T, 4><<<grid, 256, 0, c.s>>>(X, n, (int)m, Sd_, n);
                    else if (m <= 8) tri_right_inplace<T, 8><<<grid, 256, 0, c.s>>>(X, n, (int)m, Sd_, n);
                    else if (m <= 16) tri_right_inplace<T, 16><<<grid, 256, 0, c.s>>>(X, n, (int)m, Sd_, n);
                    else tri_right_inplace<T, 24><<<grid, 256, 0, c.s>>>(X, n, (int)m, Sd_, n);
                    c.check_launch();
                };
                apply(Kt);
                apply(Ut);
                c.sync();  // hS is read by the copy above
                if (kappa <= 20.0) break;  // this pass left O(kappa^2 eps) of non-orthogonality
            }
            if (ok) return;
            ++stats_rhs_cgs_fallback;
        }
        double* coef = c.sc(6);
        double* nrm = c.sc(7);
        for (long t = 0; t < m; ++t) {
            T* kt = Kt + (size_t)t * n;
            T* ut = Ut + (size_t)t * n;
            if (t > 0) {
                cgs2<T, false>(c, Kt, n, t, kt, kt, n, coef, c.sc(4), c.sc(5));
                ts_N_launch<T>(c, Ut, n, t, ut, ut, n, coef);
            }
            dbg_sum(" frs cgs kt", kt, n, c.s);
            dbg_sum(" frs coef", coef, 2 * t, c.s);
            launch_norms<T>(c, kt, n, nrm);
            dbg_sum(" frs nrm", nrm, 3, c.s);
            launch_scale<T>(c, kt, kt, n, nrm, 1);
            launch_scale<T>(c, ut, ut, n, nrm, 1);
        }
    }

    // raw column append (no image factorisation): the per-RHS-only comparator
    void append_raw(const T* y, uint8_t marker) {
        reserve(cols + 1);
        CK(cudaMemcpyAsync(Vp() + (size_t)cols * n, y, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->s));
        ++cols;
        markers.push_back(marker);
    }

    bool append(const T* y, const T* z, uint8_t marker) {
        if (cap > 0 && cols >= cap) return false;
        reserve(cols + 1);
        const long j = cols;
        CK(cudaMemcpyAsync(Vp() + (size_t)j * n, y, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->s));
        if (!factor_image(j, Vp() + (size_t)j * n, z, true)) return false;
        ++cols;
        markers.push_back(marker);
        return true;
    }

    // coords w = K^H b for b = val * e_idx (row gather), device out (cols*W)
    void coords_single(long idx, double val, double* w) {
        if (cols == 0) return;
        row_gather<T, true><<<(int)((cols + 255) / 256), 256, 0, ctx->s>>>(Kp(), n, (int)cols, idx, val, w);
        ctx->check_launch();
    }
};

struct BasisHandle {
    Ctx* ctx;
    int dtype;
    std::unique_ptr<DevBasis<double>> r;
    std::unique_ptr<DevBasis<cplx>> c;
};

// process_system (basis.cpp:157-207)
struct LogRow {
    int system, rhs;
    double init_relres;
    int iterations;
    bool appended;
};

// Host wall-clock phase accounting of process_system (ROMDOT_VERBOSE>=1);
// every phase ends in a stream sync already, so this adds no device syncs.
struct PhaseTimer {
    double t[8] = {0};
    std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    void lap(int k) {
        const auto now = std::chrono::steady_clock::now();
        t[k] += std::chrono::duration<double, std::milli>(now - last).count();
        last = now;
    }
};

template <class T>
void process_system(DevBasis<T>& gb, DevOp& op, long nrhs, const long* bidx, const double* bval, double tol,
                    int system_index, long maxit, T* Xdev, std::vector<LogRow>& log, long& inner_its,
                    long& appends) {
    Ctx& c = *gb.ctx;
    const long n = gb.n;
    if (maxit <= 0) maxit = 2 * n;
    PhaseTimer pt;
    const bool timing = verbose() >= 1;
    auto lap = [&](int k) {
        if (timing) {
            c.sync();
            pt.lap(k);
        }
    };
    gb.refresh(op);
    lap(0);
    VLOG(1, "system %d: refresh done (cols %ld, block %ld seq %ld second-pass %ld, rhs-space second passes %ld)",
         system_index, gb.cols, gb.stats_block_refresh, gb.stats_seq_refresh, gb.stats_second_pass,
         gb.stats_rhs_second_pass);
    long cspace = 1;
    for (const auto& sp : gb.spaces) cspace = std::max(cspace, (long)sp.size() + 1);
    dbg_sum("refresh K", gb.Kp(), gb.n * gb.cols, c.s);
    dbg_sum("refresh W", gb.Wp(), gb.n * gb.cols, c.s);
    gb.factor_eig_block(op, cspace);
    lap(1);
    dbg_sum("eig Kr", gb.Kr.template as<T>(), gb.n * gb.ku, c.s);
    dbg_sum("eig Ur", gb.Ur.template as<T>(), gb.n * gb.ku, c.s);
    log.clear();
    inner_its = 0;
    appends = 0;
    // ---- batched global check (basis.cpp:171-172 for every RHS at once) ----
    // b_j = val_j e_{idx_j}: K_old^H B is a row gather; R_all = B - K_old K_old^H B
    // is one tall GEMM per system; per RHS only the columns appended during the
    // system are projected out of R_all[:, j].
    const long r0 = gb.cols;
    using DB = DevBasis<T>;
    DevBuf &idxd = gb.ps_idx, &vald = gb.ps_val, &Wc = gb.ps_Wc, &Rall = gb.ps_Rall, &Coef = gb.ps_Coef,
           &Cpk = gb.ps_Cpk, &rjbuf = gb.ps_rj, &wn = gb.ps_wn, &ybuf = gb.ps_y, &gbuf = gb.ps_g, &imbuf = gb.ps_im;
    DB::grow_to(idxd, sizeof(long) * nrhs);
    DB::grow_to(vald, sizeof(double) * nrhs);
    CK(cudaMemcpyAsync(idxd.p, bidx, sizeof(long) * nrhs, cudaMemcpyHostToDevice, c.s));
    CK(cudaMemcpyAsync(vald.p, bval, sizeof(double) * nrhs, cudaMemcpyHostToDevice, c.s));
    const long npad = padded_rows(n);
    DB::grow_to(Rall, sizeof(T) * npad * nrhs);
    CK(cudaMemsetAsync(Rall.p, 0, sizeof(T) * npad * nrhs, c.s));
    if (r0 > 0) {
        DB::grow_to(Wc, sizeof(T) * r0 * nrhs);
        row_gather_multi<T, true><<<c.grid_for(r0 * nrhs, 256, 4), 256, 0, c.s>>>(
            gb.Kp(), n, 0, (int)r0, idxd.template as<long>(), vald.template as<double>(), (int)nrhs, -1.0,
            Wc.template as<T>(), r0);
        c.check_launch();
        gemm<T, false>(c, gb.Kp(), n, r0, Wc.template as<T>(), nrhs, nullptr, 0, Rall.template as<T>(), npad, n,
                       false);
    }
    scatter_add_rhs<T><<<(int)((nrhs + 127) / 128), 128, 0, c.s>>>(Rall.template as<T>(), npad, idxd.template as<long>(),
                                                                   vald.template as<double>(), (int)nrhs);
    c.check_launch();
    dbg_sum("Rall", Rall.template as<T>(), npad * nrhs, c.s);
    // deferred solution assembly X = G + W Coef (solve_projected, basis.cpp:110-112)
    const long capc = std::max(gb.capcols, r0 + nrhs + 1);
    if (Xdev) {
        DB::grow_to(Coef, sizeof(T) * capc * nrhs);
        CK(cudaMemsetAsync(Coef.p, 0, sizeof(T) * capc * nrhs, c.s));
    }
    for (DevBuf* b : {&rjbuf, &ybuf, &gbuf, &imbuf}) {  // zero-tailed (TMA passes)
        DB::grow_to(*b, sizeof(T) * npad);
        CK(cudaMemsetAsync(b->p, 0, sizeof(T) * npad, c.s));
    }
    DB::grow_to(wn, sizeof(T) * (nrhs + 8));
    lap(2);
    // ---- independent tail (candidate cap reached: no right-hand side appends any more, so
    // none changes the state another one starts from; basis.cpp:168-205 with append() == false).
    // Their global checks run back to back and their correction solves BD_M at a time with
    // the system's eigen block streamed once for all of them (bcg_defl.cuh). A slot that
    // finishes is refilled with the next pending right-hand side.
    auto batched_tail = [&](long j0) {
        if (!gb.bd) gb.bd = std::make_unique<BatchedDeflated<T>>();
        BatchedDeflated<T>& bd = *gb.bd;
        constexpr int M = BatchedDeflated<T>::M;
        const long rcur = gb.cols, nt = nrhs - j0;
        long tmax = 0;
        for (long j = j0; j < nrhs; ++j) tmax = std::max(tmax, (long)gb.spaces[j].size() - gb.ku);
        if (gb.hook)
            for (long j = j0; j < nrhs; ++j) {
                c.sync();
                if (gb.hook(gb.hook_user, system_index, j) != 0)
                    throw SolverError("process_system: rhs hook aborted at system " + std::to_string(system_index) +
                                      ", rhs " + std::to_string(j));
            }
        DB::grow_to(gb.ps_nrm, sizeof(double) * 8 * nt);
        double* nrmd = gb.ps_nrm.template as<double>();
        for (long j = j0; j < nrhs; ++j) {
            T* rhs = Rall.template as<T>() + (size_t)j * npad;
            if (rcur > r0) {  // project out this system's appended columns (in place)
                DB::grow_to(wn, sizeof(T) * (rcur - r0));
                row_gather_multi<T, true><<<c.grid_for(rcur - r0, 256, 1), 256, 0, c.s>>>(
                    gb.Kp(), n, (int)r0, (int)(rcur - r0), idxd.template as<long>() + j,
                    vald.template as<double>() + j, 1, 1.0, wn.template as<T>(), rcur - r0);
                c.check_launch();
                global_N<T>(c, gb.Kp() + (size_t)r0 * n, n, rcur - r0, rhs, rhs, n, (const double*)wn.p);
            }
            launch_norms<T>(c, rhs, n, nrmd + 8 * (j - j0));
            if (Xdev) {
                row_gather_multi<T, true><<<c.grid_for(rcur, 256, 1), 256, 0, c.s>>>(
                    gb.Kp(), n, 0, (int)rcur, idxd.template as<long>() + j, vald.template as<double>() + j, 1, -1.0,
                    Coef.template as<T>() + (size_t)j * capc, capc);
                c.check_launch();
            }
        }
        std::vector<double> hn(8 * nt);
        CK(cudaMemcpyAsync(hn.data(), nrmd, sizeof(double) * 8 * nt, cudaMemcpyDeviceToHost, c.s));
        c.sync();
        lap(2);
        std::vector<LogRow> rows;
        std::vector<long> pending;
        for (long j = j0; j < nrhs; ++j) {
            rows.push_back(LogRow{system_index, (int)j, std::sqrt(hn[8 * (j - j0)]) / std::fabs(bval[j]), 0, false});
            if (rows.back().init_relres <= tol) {
                if (Xdev) CK(cudaMemsetAsync(Xdev + (size_t)j * n, 0, sizeof(T) * n, c.s));
            } else {
                pending.push_back(j);
            }
        }
        if (!pending.empty()) {
            // longest first: the iteration count grows with the initial residual, and the last
            // slots to drain run alone (results do not depend on the order; rows stay in RHS order)
            std::stable_sort(pending.begin(), pending.end(), [&](long a, long b) {
                return rows[a - j0].init_relres > rows[b - j0].init_relres;
            });
            bd.begin_system(c, op.d, gb.Kr.template as<T>(), gb.ku, tmax);
            long slot_rhs[M];
            for (int m = 0; m < M; ++m) slot_rhs[m] = -1;
            size_t next = 0;
            int active = 0;
            double t_space = 0, t_gram = 0, t_load = 0, t_fin = 0, t_iter = 0;  // ROMDOT_VERBOSE >= 1
            auto tick = [&](double& acc, auto&& fn) {
                if (!timing) {
                    fn();
                    return;
                }
                c.sync();
                const auto a = std::chrono::steady_clock::now();
                fn();
                c.sync();
                acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
            };
            auto fill = [&](int m) {
                if (next >= pending.size()) return false;
                const long j = pending[next++];
                auto& idx = gb.spaces[j];
                tick(t_space, [&] { gb.factor_rhs_space(op, idx); });
                const T* Gsp = nullptr;
                tick(t_gram, [&] { Gsp = gb.space_gram((long)idx.size()); });
                tick(t_load, [&] {
                    bd.load(m, gb.Kr.template as<T>(), gb.Ur.template as<T>(), (long)idx.size(), Gsp,
                            Rall.template as<T>() + (size_t)j * npad, kInnerSafety * tol, maxit, std::fabs(bval[j]));
                });
                slot_rhs[m] = j;
                ++active;
                return true;
            };
            const int mslots = batch_width();
            for (int m = 0; m < mslots; ++m) fill(m);
            long steps = 0, slot_steps = 0;
            while (active > 0) {
                steps += batch_steps();
                slot_steps += (long)active * batch_steps();
                const CGState* hs = nullptr;
                tick(t_iter, [&] {
                    bd.iterate(op.d, batch_steps());
                    hs = bd.poll();
                });
                for (int m = 0; m < M; ++m) {
                    const long j = slot_rhs[m];
                    if (j < 0 || !hs[m].done) continue;
                    if (!hs[m].converged)
                        throw SolverError("process_system: correction solve failed at system " +
                                          std::to_string(system_index) + ", rhs " + std::to_string(j));
                    rows[j - j0].iterations = hs[m].it;
                    inner_its += hs[m].it;
                    T* Gj = Xdev ? Xdev + (size_t)j * n : gbuf.template as<T>();
                    tick(t_fin, [&] {
                        bd.finish(m, op, gb.Kr.template as<T>(), gb.Ur.template as<T>(), Gj, nullptr,
                                  imbuf.template as<T>());
                    });
                    slot_rhs[m] = -1;
                    --active;
                    ++gb.stats_batched_rhs;
                    if (!fill(m)) bd.release(m);
                }
            }
            VLOG(1,
                 "system %d batched tail: %zu solves, %ld steps of %d slots, %.2f slots busy on average | ms: spaces "
                 "%.1f space-gram %.1f load %.1f iterate %.1f (%.3f per step) finish %.1f",
                 system_index, pending.size(), steps, M, steps ? (double)slot_steps / steps : 0.0, t_space, t_gram,
                 t_load, t_iter, steps ? t_iter / steps : 0.0, t_fin);
        }
        lap(4);
        for (const LogRow& row : rows) {
            VLOG(2, "system %d rhs %d: init_relres %.3e its %d appended 0 cols %ld (batched)", system_index, row.rhs,
                 row.init_relres, row.iterations, gb.cols);
            log.push_back(row);
        }
    };
    for (long j = 0; j < nrhs; ++j) {
        if (batch_slots() && c.solver == 0 && use_one_pass_projection() && gb.cap > 0 && gb.cols >= gb.cap &&
            nrhs - j >= 2) {
            long tmax = 0;
            for (long q = j; q < nrhs; ++q) tmax = std::max(tmax, (long)gb.spaces[q].size() - gb.ku);
            if (BatchedDeflated<T>::supported(gb.ku, tmax)) {
                batched_tail(j);
                break;
            }
        }
        if (gb.hook) {
            c.sync();
            if (gb.hook(gb.hook_user, system_index, j) != 0)
                throw SolverError("process_system: rhs hook aborted at system " + std::to_string(system_index) +
                                  ", rhs " + std::to_string(j));
        }
        const double bnorm = std::fabs(bval[j]);
        const long rcur = gb.cols;
        const T* rhs = Rall.template as<T>() + (size_t)j * npad;
        if (rcur > r0) {  // project out this system's appended columns
            DB::grow_to(wn, sizeof(T) * (rcur - r0));
            row_gather_multi<T, true><<<c.grid_for(rcur - r0, 256, 1), 256, 0, c.s>>>(
                gb.Kp(), n, (int)r0, (int)(rcur - r0), idxd.template as<long>() + j, vald.template as<double>() + j, 1,
                1.0, wn.template as<T>(), rcur - r0);
            c.check_launch();
            global_N<T>(c, gb.Kp() + (size_t)r0 * n, n, rcur - r0, rhs, rjbuf.template as<T>(), n,
                        (const double*)wn.p);
            rhs = rjbuf.template as<T>();
        }
        double* nrm = c.sc(3);
        launch_norms<T>(c, rhs, n, nrm);
        double h;
        CK(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        if (Xdev) {  // Coef[:rcur, j] = -K^H b_j (negated for the final Y - X M GEMM)
            row_gather_multi<T, true><<<c.grid_for(rcur, 256, 1), 256, 0, c.s>>>(
                gb.Kp(), n, 0, (int)rcur, idxd.template as<long>() + j, vald.template as<double>() + j, 1, -1.0,
                Coef.template as<T>() + (size_t)j * capc, capc);
            c.check_launch();
        }
        c.sync();
        lap(2);
        LogRow row{system_index, (int)j, std::sqrt(h) / bnorm, 0, false};
        T* Gj = Xdev ? Xdev + (size_t)j * n : gbuf.template as<T>();
        if (row.init_relres <= tol) {
            if (Xdev) CK(cudaMemsetAsync(Gj, 0, sizeof(T) * n, c.s));
        } else {
            auto& idx = gb.spaces[j];
            const long cj = (long)idx.size();
            dbg_sum("rhs", rhs, n, c.s);
            gb.factor_rhs_space(op, idx);
            lap(3);
            dbg_sum("space K", gb.Kr.template as<T>(), n * cj, c.s);
            dbg_sum("space U", gb.Ur.template as<T>(), n * cj, c.s);
            const T* Gsp = use_one_pass_projection() && c.solver == 0 ? gb.space_gram(cj) : nullptr;
            SolveOut so = recycled_solve<T>(c, op, gb.Ur.template as<T>(), gb.Kr.template as<T>(), cj, rhs,
                                         kInnerSafety * tol, maxit, bnorm, Gj, ybuf.template as<T>(),
                                         imbuf.template as<T>(), gb.ws, false, true, Gsp);
            if (!so.converged)
                throw SolverError("process_system: correction solve failed at system " +
                                  std::to_string(system_index) + ", rhs " + std::to_string(j));
            lap(4);
            row.iterations = so.iterations;
            inner_its += so.iterations;
            dbg_sum("y", ybuf.template as<T>(), n, c.s);
            dbg_sum("image", imbuf.template as<T>(), n, c.s);
            if (gb.append(ybuf.template as<T>(), imbuf.template as<T>(), kColCorrection)) {
                idx.push_back((int)(gb.cols - 1));
                row.appended = true;
                ++appends;
                dbg_sum("appended K col", gb.Kp() + (size_t)(gb.cols - 1) * n, n, c.s);
                if (!DevBasis<T>::lazy_w())  // lazy W: the column is formed later (materialize_W)
                    dbg_sum("appended W col", gb.Wp() + (size_t)(gb.cols - 1) * n, n, c.s);
            }
            lap(5);
        }
        VLOG(2, "system %d rhs %ld: init_relres %.3e its %d appended %d cols %ld", system_index, j, row.init_relres,
             row.iterations, (int)row.appended, gb.cols);
        log.push_back(row);
    }
    if (Xdev && gb.cols > 0) {
        const long rf = gb.cols;
        DB::grow_to(Cpk, sizeof(T) * rf * nrhs);
        CK(cudaMemcpy2DAsync(Cpk.p, sizeof(T) * rf, Coef.p, sizeof(T) * capc, sizeof(T) * rf, nrhs,
                             cudaMemcpyDeviceToDevice, c.s));
        dbg_sum("X corrections", Xdev, n * nrhs, c.s);
        dbg_sum("X coefficients", Cpk.template as<T>(), rf * nrhs, c.s);
        gb.materialize_W();
        dbg_sum("X W", gb.Wp(), n * rf, c.s);
        gemm<T, true>(c, gb.Wp(), n, rf, Cpk.template as<T>(), nrhs, Xdev, n, Xdev, n, n, false);
        dbg_sum("X assembled", Xdev, n * nrhs, c.s);
    }
    c.sync();
    dbg_flush(c.s);
    lap(6);
    VLOG(1,
         "system %d phases (ms): refresh %.1f eig-block %.1f checks %.1f rhs-spaces %.1f solves %.1f appends %.1f "
         "X-assembly %.1f | %ld its",
         system_index, pt.t[0], pt.t[1], pt.t[2], pt.t[3], pt.t[4], pt.t[5], pt.t[6], inner_its);
}

// BaselinePerRhsRecycler::solve_system (basis.cpp:221-264) on the device:
// the comparator that recycles only each RHS's own space U_j = [U0, X0_j, own
// directions] -- no global check, no cross-RHS sharing. Storage is a raw
// DevBasis (V + index lists). Per system the shared eigen block is factored
// once (factor_eig_block); per RHS the trailing columns (factor_rhs_space),
// then the recycled CG / COCG at tol (not 0.25 tol, :244) on b_j itself: its
// output g = U K^T b + (y - U K^T A y) is z0 + correction (:249), its first
// residual is init_relres (:236-239), and y_m is appended when it iterated.
template <class T>
void per_rhs_solve_system(DevBasis<T>& gb, DevOp& op, long nrhs, const long* bidx, const double* bval, double tol,
                          int system_index, long maxit, T* Xdev, std::vector<LogRow>& log, long& inner_its,
                          long& appends) {
    Ctx& c = *gb.ctx;
    const long n = gb.n;
    if (maxit <= 0) maxit = 2 * n;
    if (nrhs != (long)gb.spaces.size()) throw ConfigError("baseline recycling: rhs count mismatch");
    long cspace = 1;
    for (const auto& sp : gb.spaces) cspace = std::max(cspace, (long)sp.size());
    gb.factor_eig_block(op, cspace);
    log.clear();
    inner_its = 0;
    appends = 0;
    const long npad = padded_rows(n);
    DevBuf rhsb, ybuf, imbuf, gbuf;
    for (DevBuf* b : {&rhsb, &ybuf, &imbuf, &gbuf}) {  // zero-tailed (TMA passes)
        b->ensure(sizeof(T) * npad);
        CK(cudaMemsetAsync(b->p, 0, sizeof(T) * npad, c.s));
    }
    const T zero = Sc<T>::zero();
    for (long j = 0; j < nrhs; ++j)
        if (bidx[j] < 0 || bidx[j] >= n) throw ConfigError("baseline recycling: rhs index out of range");
    // Every right-hand side of this comparator is independent of the others (its space holds
    // its own directions only and nothing is shared, basis.cpp:221-264), so the solves run
    // BD_M at a time with the eigen block streamed once for all of them (bcg_defl.cuh). The
    // new directions are appended afterwards in right-hand-side order, so V and the index
    // lists are the ones the one-at-a-time loop below leaves.
    long tmax = 0;
    for (const auto& sp : gb.spaces) tmax = std::max(tmax, (long)sp.size() - gb.ku);
    if (batch_slots() && c.solver == 0 && use_one_pass_projection() && nrhs >= 2 &&
        BatchedDeflated<T>::supported(gb.ku, tmax)) {
        using DB = DevBasis<T>;
        if (!gb.bd) gb.bd = std::make_unique<BatchedDeflated<T>>();
        BatchedDeflated<T>& bd = *gb.bd;
        constexpr int M = BatchedDeflated<T>::M;
        DB::grow_to(gb.ps_Rall, sizeof(T) * n * nrhs);  // the y_m of every right-hand side, kept until the appends
        T* Yall = gb.ps_Rall.template as<T>();
        bd.begin_system(c, op.d, gb.Kr.template as<T>(), gb.ku, tmax);
        std::vector<LogRow> rows(nrhs);
        long slot_rhs[M];
        for (int m = 0; m < M; ++m) slot_rhs[m] = -1;
        long next = 0;
        int active = 0;
        T* rhs = rhsb.template as<T>();
        auto fill = [&](int m) {
            if (next >= nrhs) return false;
            const long j = next++;
            const T bv = Sc<T>::from(bval[j]);
            CK(cudaMemcpyAsync(rhs + bidx[j], &bv, sizeof(T), cudaMemcpyHostToDevice, c.s));
            auto& idx = gb.spaces[j];
            gb.factor_rhs_space(op, idx);
            const T* Gsp = gb.space_gram((long)idx.size());
            bd.load(m, gb.Kr.template as<T>(), gb.Ur.template as<T>(), (long)idx.size(), Gsp, rhs, tol, maxit,
                    std::fabs(bval[j]));
            CK(cudaMemcpyAsync(rhs + bidx[j], &zero, sizeof(T), cudaMemcpyHostToDevice, c.s));
            c.sync();  // bv is a stack value
            slot_rhs[m] = j;
            ++active;
            return true;
        };
        const int mslots = batch_width();
        for (int m = 0; m < mslots; ++m) fill(m);
        while (active > 0) {
            bd.iterate(op.d, batch_steps());
            const CGState* hs = bd.poll();
            for (int m = 0; m < M; ++m) {
                const long j = slot_rhs[m];
                if (j < 0 || !hs[m].done) continue;
                if (!hs[m].converged)
                    throw SolverError("baseline recycling: solve failed at system " + std::to_string(system_index) +
                                      ", rhs " + std::to_string(j));
                rows[j] = LogRow{system_index, (int)j, bd.h0h[m], hs[m].it, false};
                T* Gj = Xdev ? Xdev + (size_t)j * n : gbuf.template as<T>();
                bd.finish(m, op, gb.Kr.template as<T>(), gb.Ur.template as<T>(), Gj, Yall + (size_t)j * n,
                          imbuf.template as<T>());
                slot_rhs[m] = -1;
                --active;
                ++gb.stats_batched_rhs;
                if (!fill(m)) bd.release(m);
            }
        }
        for (long j = 0; j < nrhs; ++j) {
            if (rows[j].iterations > 0) {
                gb.append_raw(Yall + (size_t)j * n, kColCorrection);
                gb.spaces[j].push_back((int)(gb.cols - 1));
                rows[j].appended = true;
                ++appends;
                inner_its += rows[j].iterations;
            }
            log.push_back(rows[j]);
        }
        c.sync();
        return;
    }
    for (long j = 0; j < nrhs; ++j) {
        const double bnorm = std::fabs(bval[j]);
        const T bv = Sc<T>::from(bval[j]);
        T* rhs = rhsb.template as<T>();
        CK(cudaMemcpyAsync(rhs + bidx[j], &bv, sizeof(T), cudaMemcpyHostToDevice, c.s));
        auto& idx = gb.spaces[j];
        const long cj = (long)idx.size();
        gb.factor_rhs_space(op, idx);
        T* Gj = Xdev ? Xdev + (size_t)j * n : gbuf.template as<T>();
        const T* Gsp = use_one_pass_projection() && c.solver == 0 ? gb.space_gram(cj) : nullptr;
        SolveOut so = recycled_solve<T>(c, op, gb.Ur.template as<T>(), gb.Kr.template as<T>(), cj, rhs, tol, maxit, bnorm,
                                     Gj, ybuf.template as<T>(), imbuf.template as<T>(), gb.ws, true, true, Gsp);
        CK(cudaMemcpyAsync(rhs + bidx[j], &zero, sizeof(T), cudaMemcpyHostToDevice, c.s));
        c.sync();  // bv / zero are host stack values
        if (!so.converged)
            throw SolverError("baseline recycling: solve failed at system " + std::to_string(system_index) +
                              ", rhs " + std::to_string(j));
        LogRow row{system_index, (int)j, so.hist.empty() ? 0.0 : so.hist[0], so.iterations, false};
        if (so.iterations > 0) {
            gb.append_raw(ybuf.template as<T>(), kColCorrection);
            idx.push_back((int)(gb.cols - 1));
            row.appended = true;
            ++appends;
            inner_its += so.iterations;
        }
        log.push_back(row);
    }
    c.sync();
}

// ------------------------------------------------------------------ RRQR ---
// Rank-revealing compression of the candidate basis (BASELINE RRQR, the
// reference's truncation rule at acceptance.cpp:378-383): column-pivoted QR
// computed as recursive block-pivoted CholQR on the device.
//   level: G = Z^H Z (device Gram) -> greedy pivoted Cholesky on the device
//   (pivot = largest residual column norm, the QRCP rule) accepting pivots
//   within 8 decades of the level's largest residual norm^2 -> Q_P =
//   CholQR2(Z_P) -> Z_rest <- (I - Q_P Q_P^H)^2 Z_rest (explicit BCGS2) ->
//   next level on the deflated columns. The explicit deflation keeps every
//   level's Gram accurate relative to its own scale, so residual norms down
//   to ~1e-14 of the first are resolved (the Gram alone stops near 1e-8).
// rank = #{R_kk > tol * R_00}; Q (n x rank) spans the retained columns.
template <class T>
long rrqr_dev(Ctx& c, long n, long m, const T* A, double tol, bool normalize, std::vector<long>& perm,
              std::vector<double>& rdiag_out, DevBuf& Qout, T* inplace = nullptr) {
    constexpr int W = Sc<T>::W;
    const long ld = n;
    DevBuf Zown, Zb, G, Sp, Sinv, Rrow, pivd, rdg, infod, work, tmp, nrm, idxd, Zs[2];
    // Zcur: the working set (the caller's buffer when in place at level 0, then
    // compacted copies in Zs[0] / Zs[1])
    T* Zcur = inplace;
    if (!inplace) {
        Zown.ensure(sizeof(T) * n * std::max(1L, m));
        CK(cudaMemcpyAsync(Zown.p, A, sizeof(T) * n * m, cudaMemcpyDeviceToDevice, c.s));
        Zcur = Zown.template as<T>();
    }
    nrm.ensure(sizeof(double) * std::max(1L, 2 * m));
    if (normalize && m > 0) {
        for (long j0 = 0; j0 < m; j0 += 1024) {
            const long cc = std::min(1024L, m - j0);
            col_norms<T><<<c.grid_for(n, 256, 2), 256, sizeof(double) * cc, c.s>>>(Zcur + j0 * ld, ld,
                                                                                   (int)cc, n, c.red(),
                                                                                   nrm.template as<double>() + j0);
            c.check_launch();
        }
        scale_columns<T><<<dim3(c.grid_for(n, 256, 1), (unsigned)m), 256, 0, c.s>>>(Zcur, ld, (int)m, n,
                                                                                   nrm.template as<double>());
        c.check_launch();
    }
    Qout.ensure(sizeof(T) * n * std::max(1L, m));
    idxd.ensure(sizeof(int) * std::max(1L, m));
    int zs = 0;  // next free compaction buffer
    // gather columns cols (local indices of Zcur) into a fresh compaction buffer
    auto compact = [&](const std::vector<int>& cols) -> T* {
        const long k = (long)cols.size();
        DevBuf& dst = Zs[zs];
        zs ^= 1;
        if (dst.bytes < sizeof(T) * n * k) dst.ensure(sizeof(T) * n * k);
        CK(cudaMemcpyAsync(idxd.p, cols.data(), sizeof(int) * k, cudaMemcpyHostToDevice, c.s));
        gather_columns<T><<<dim3(c.grid_for(n, 256, 1), (unsigned)k), 256, 0, c.s>>>(
            Zcur, ld, idxd.template as<int>(), (int)k, n, dst.template as<T>(), ld);
        c.check_launch();
        c.sync();  // cols is host memory of the caller's frame
        return dst.template as<T>();
    };
    auto col_norms_host = [&](const T* X, long k, std::vector<double>& out) {
        out.resize(k);
        for (long j0 = 0; j0 < k; j0 += 1024) {
            const long cc = std::min(1024L, k - j0);
            col_norms<T><<<c.grid_for(n, 256, 2), 256, sizeof(double) * cc, c.s>>>(
                X + j0 * ld, ld, (int)cc, n, c.red(), nrm.template as<double>() + j0);
            c.check_launch();
        }
        CK(cudaMemcpyAsync(out.data(), nrm.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c.s));
        c.sync();
    };
    std::vector<long> remaining(m);  // original column of each working-set column
    for (long j = 0; j < m; ++j) remaining[j] = j;
    perm.clear();
    rdiag_out.clear();
    std::vector<long> dropped;  // residual norm <= tol * R_00: can never be a pivot
    double r00 = -1.0;
    long rank = 0;
    bool done = false;
    int level = 0;
    long second_passes = 0;
    PhaseTimer pt;  // ROMDOT_VERBOSE >= 1: per-phase wall time (adds syncs)
    const bool timing = verbose() >= 1;
    auto lap = [&](int k) {
        if (timing) {
            c.sync();
            pt.lap(k);
        }
    };
    lap(7);
    while (!done && !remaining.empty()) {
        const long mr = (long)remaining.size();
        G.ensure(sizeof(T) * mr * mr);
        gram<T, true>(c, Zcur, ld, mr, Zcur, ld, mr, n, G.template as<T>(), true, work);
        lap(0);
        Rrow.ensure(sizeof(T) * mr * mr);
        pivd.ensure(sizeof(int) * mr);
        rdg.ensure(sizeof(double) * mr);
        infod.ensure(sizeof(double) * 4);
        const double stop_abs2 = r00 > 0.0 ? (tol * r00) * (tol * r00) : 0.0;
        const size_t shm = sizeof(double) * mr + sizeof(int) * mr;
        if (shm > 200 * 1024) throw ConfigError("rrqr: candidate basis too wide");
        CK(cudaFuncSetAttribute(pivoted_chol<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        pivoted_chol<T><<<1, 1024, shm, c.s>>>(G.template as<T>(), (int)mr, stop_abs2, 1e-8, pivd.template as<int>(),
                                               rdg.template as<double>(), Rrow.template as<T>(),
                                               infod.template as<double>());
        c.check_launch();
        double info[3];
        CK(cudaMemcpyAsync(info, infod.p, sizeof(info), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        const long nsel = (long)info[0];
        std::vector<int> piv(nsel);
        std::vector<double> rdl(nsel);
        if (nsel) {
            CK(cudaMemcpy(piv.data(), pivd.p, sizeof(int) * nsel, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(rdl.data(), rdg.p, sizeof(double) * nsel, cudaMemcpyDeviceToHost));
        }
        if (r00 < 0.0) r00 = nsel ? rdl[0] : 0.0;
        lap(1);
        // accept pivots above the rank threshold
        long keep = 0;
        while (keep < nsel && rdl[keep] > tol * r00) ++keep;
        for (long k = 0; k < keep; ++k) {
            perm.push_back(remaining[piv[k]]);
            rdiag_out.push_back(rdl[k]);
        }
        if (keep < nsel || info[2] > 0.5 || nsel == 0) done = true;
        T* QP = Qout.template as<T>() + rank * ld;
        if (keep > 0) {
            // Z_P (gathered, pivot order) -> Q_P = Z_P S_PP^-1, then a CholQR pass
            Zb.ensure(sizeof(T) * n * keep);
            T* ZP = Zb.template as<T>();
            CK(cudaMemcpyAsync(idxd.p, piv.data(), sizeof(int) * keep, cudaMemcpyHostToDevice, c.s));
            gather_columns<T><<<dim3(c.grid_for(n, 256, 1), (unsigned)keep), 256, 0, c.s>>>(
                Zcur, ld, idxd.template as<int>(), (int)keep, n, ZP, ld);
            c.check_launch();
            // S_PP (keep x keep upper) from Rrow rows restricted to the picked columns
            std::vector<T> Rh((size_t)keep * mr);
            CK(cudaMemcpy(Rh.data(), Rrow.p, sizeof(T) * keep * mr, cudaMemcpyDeviceToHost));
            std::vector<T> S((size_t)keep * keep, Sc<T>::zero());
            for (long kk = 0; kk < keep; ++kk)
                for (long i = 0; i <= kk; ++i) S[i + kk * keep] = Rh[(size_t)i * mr + piv[kk]];
            Sp.ensure(sizeof(T) * keep * keep);
            Sinv.ensure(sizeof(T) * keep * keep);
            CK(cudaMemcpyAsync(Sp.p, S.data(), sizeof(T) * keep * keep, cudaMemcpyHostToDevice, c.s));
            tri_inv_upper<T><<<1, 1024, 0, c.s>>>(Sp.template as<T>(), Sinv.template as<T>(), (int)keep);
            c.check_launch();
            gemm<T, false>(c, ZP, ld, keep, Sinv.template as<T>(), keep, nullptr, 0, QP, ld, n, true);
            lap(2);
            for (int pass = 0; pass < 2; ++pass) {  // CholQR2 clean-up of Q_P
                gram<T, true>(c, QP, ld, keep, QP, ld, keep, n, Sp.template as<T>(), true, work);
                CholInfo ci = chol_inv<T, true>(c, Sp.template as<T>(), Sinv.template as<T>(), keep, false);
                if (ci.bad) throw SolverError("rrqr: CholQR of the pivot block failed");
                gemm<T, false>(c, QP, ld, keep, Sinv.template as<T>(), keep, nullptr, 0, ZP, ld, n, true);
                CK(cudaMemcpyAsync(QP, ZP, sizeof(T) * n * keep, cudaMemcpyDeviceToDevice, c.s));
            }
            rank += keep;
            lap(3);
        }
        // the columns not picked at this level, compacted (out of place)
        std::vector<char> pk(mr, 0);
        for (long k = 0; k < keep; ++k) pk[piv[k]] = 1;
        std::vector<long> rest;
        std::vector<int> rest_local;
        for (long i = 0; i < mr; ++i)
            if (!pk[i]) {
                rest.push_back(remaining[i]);
                rest_local.push_back((int)i);
            }
        if (done || rest.empty()) {
            for (long v : rest) perm.push_back(v);
            break;
        }
        const long nr = (long)rest.size();
        if (keep > 0) Zcur = compact(rest_local);
        // block CGS against the new block Q_P (the working set is already
        // orthogonal to the earlier blocks); a second pass against every
        // retained direction only if some column lost more than half of its
        // norm^2 (Kahan-Parlett, as the global appends)
        std::vector<double> nb, na;
        col_norms_host(Zcur, nr, nb);
        tmp.ensure(sizeof(T) * std::max(1L, rank) * nr);
        if (keep > 0) {
            gram<T, true>(c, QP, ld, keep, Zcur, ld, nr, n, tmp.template as<T>(), false, work);
            gemm<T, true>(c, QP, ld, keep, tmp.template as<T>(), nr, Zcur, ld, Zcur, ld, n, false);
        }
        col_norms_host(Zcur, nr, na);
        bool cancel = false;
        for (long j = 0; j < nr; ++j) cancel |= na[j] < 0.5 * nb[j];
        if (cancel) {
            ++second_passes;
            gram<T, true>(c, Qout.template as<T>(), ld, rank, Zcur, ld, nr, n, tmp.template as<T>(), false, work);
            gemm<T, true>(c, Qout.template as<T>(), ld, rank, tmp.template as<T>(), nr, Zcur, ld, Zcur, ld, n,
                          false);
            col_norms_host(Zcur, nr, na);
        }
        // a column whose residual norm is <= tol * R_00 can never give R_kk >
        // tol * R_00 (deflation only shrinks it): out of the working set
        std::vector<int> live;
        std::vector<long> surv;
        const double cut = (tol * r00) * (tol * r00);
        for (long j = 0; j < nr; ++j) {
            if (na[j] > cut) {
                live.push_back((int)j);
                surv.push_back(rest[j]);
            } else {
                dropped.push_back(rest[j]);
            }
        }
        if (!live.empty() && (long)live.size() < nr) Zcur = compact(live);
        lap(4);
        VLOG(1, "rrqr level %d: %ld columns, %ld picked, %ld kept, rank %ld, %ld live after deflation%s", level, mr,
             nsel, keep, rank, (long)live.size(), cancel ? " (second pass)" : "");
        remaining = surv;
        ++level;
        if (level > 64) throw SolverError("rrqr: too many levels");
    }
    for (long v : dropped) perm.push_back(v);
    for (long j = 0; j < m; ++j)
        if (std::find(perm.begin(), perm.end(), j) == perm.end()) perm.push_back(j);
    VLOG(1, "rrqr phases (ms): gram %.1f pivoted-chol %.1f pivot-block %.1f cholqr2 %.1f deflation %.1f | "
            "n %ld m %ld rank %ld levels %d second passes %ld", pt.t[0], pt.t[1], pt.t[2], pt.t[3], pt.t[4], n, m,
         rank, level + 1, second_passes);
    (void)W;
    return rank;
}

}  // namespace rd

// ================================================================ C ABI ===
using namespace rd;

// ------------------------------------------------------- reduced model ---
// ReducedModel (src/rom.cpp:9-67) on the device, one-sided bilinear projection
// onto V: A_r(p) = V^T A(p) V assembled per call by a
// multi-column stencil pass + Gram in 64-column chunks (variable D makes the
// reference's affine A*_r + V^T diag(mu) V split unavailable; the cost is the
// same O(n r^2)), symmetrised, LU with partial pivoting, multi-RHS solve.
namespace rd {
template <class T> struct DevRom {
    Ctx* ctx = nullptr;
    long n = 0, r = 0;
    DevBuf own;  // owned copy when V came from the host; else V is borrowed
    const T* V = nullptr;
    DevBuf E, Ar, AV, piv, info, B, Cr, WY, WZ, G, Sinv, gwork, ix, vx, Pd;
    static constexpr long kChunk = 64;

    void init(Ctx& c, long n_, long r_, const void* Vin, int where) {
        ctx = &c;
        n = n_;
        r = r_;
        if (r <= 0 || n <= 0 || r > n) throw ConfigError("rom: need 0 < r <= n");
        if (r > 2048) throw ConfigError("rom: order limited to 2048");
        if (where == 1) {
            V = static_cast<const T*>(Vin);
        } else {
            own.ensure(sizeof(T) * n * r);
            CK(cudaMemcpyAsync(own.p, Vin, sizeof(T) * n * r, cudaMemcpyHostToDevice, c.s));
            V = own.template as<T>();
        }
        // E_r = V^T V (rom.cpp:11); the rank check is the Cholesky of the
        // Hermitian Gram V^H V (= V^T V for real bases, rom.cpp:12-14)
        E.ensure(sizeof(T) * r * r);
        gram<T, false>(c, V, n, r, V, n, r, n, E.template as<T>(), true, gwork);
        G.ensure(sizeof(T) * r * r);
        Sinv.ensure(sizeof(T) * r * r);
        gram<T, true>(c, V, n, r, V, n, r, n, G.template as<T>(), true, gwork);
        const CholInfo ci = chol_inv<T, true>(c, G.template as<T>(), Sinv.template as<T>(), r, false);
        if (ci.bad) throw SolverError("rom: basis is numerically rank deficient (E_r not SPD)");
    }

    // A_r = sym(V^T A V) into Ar (device, ld r)
    void reduced_system(const OpDev& op) {
        Ctx& c = *ctx;
        if (op.n != n) throw ConfigError("rom: operator dimension mismatch");
        Ar.ensure(sizeof(T) * r * r);
        AV.ensure(sizeof(T) * n * std::min(r, kChunk));
        T* A = Ar.template as<T>();
        for (long c0 = 0; c0 < r; c0 += kChunk) {
            const long cw = std::min(kChunk, r - c0);
            launch_stencil<T>(c, op, V + (size_t)c0 * n, n, nullptr, AV.template as<T>(), n, cw);
            gram<T, false>(c, V, n, r, AV.template as<T>(), n, cw, n, A + (size_t)c0 * r, false, gwork);
        }
        rom_symmetrize<T><<<c.grid_for(r * r, 256, 2), 256, 0, c.s>>>(A, (int)r);
        c.check_launch();
    }

    // in-place LU of Ar (partial pivoting); throws on an exactly singular pivot
    void factor() {
        Ctx& c = *ctx;
        piv.ensure(sizeof(int) * r);
        info.ensure(sizeof(int));
        CK(cudaMemsetAsync(info.p, 0, sizeof(int), c.s));
        T* A = Ar.template as<T>();
        for (long k = 0; k < r; ++k) {
            lu_pivot_col<T><<<1, 1024, 0, c.s>>>(A, (int)r, (int)k, piv.template as<int>(), info.template as<int>());
            c.check_launch();
            const long m = r - k - 1;
            if (m > 0) {
                lu_update<T><<<c.grid_for(m * m, 256, 4), 256, 0, c.s>>>(A, (int)r, (int)k);
                c.check_launch();
            }
        }
        int h = 0;
        CK(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        if (h) throw SolverError("rom: reduced system factorization failed");
    }

    void solve(T* X, long nrhs) {
        Ctx& c = *ctx;
        if (nrhs <= 0) return;
        const size_t smem = sizeof(T) * r;
        lu_solve<T><<<(unsigned)nrhs, 512, smem, c.s>>>(Ar.template as<T>(), (int)r, piv.template as<int>(), X, r);
        c.check_launch();
    }

    // B_r = V^T B for a layout block with one nonzero per column (grid.cpp:146-158)
    void gather(const long* idx, const double* val, long m, T* out) {
        Ctx& c = *ctx;
        if (m <= 0) return;
        ix.ensure(sizeof(long) * m);
        vx.ensure(sizeof(double) * m);
        CK(cudaMemcpyAsync(ix.p, idx, sizeof(long) * m, cudaMemcpyHostToDevice, c.s));
        CK(cudaMemcpyAsync(vx.p, val, sizeof(double) * m, cudaMemcpyHostToDevice, c.s));
        for (long j = 0; j < m; ++j)
            if (idx[j] < 0 || idx[j] >= n) throw ConfigError("rom: layout index out of range");
        row_gather_multi<T, false><<<c.grid_for(r * m, 256, 4), 256, 0, c.s>>>(
            V, n, 0, (int)r, ix.template as<long>(), vx.template as<double>(), (int)m, 1.0, out, r);
        c.check_launch();
        c.sync();  // ix / vx are reused by the next gather
    }

    // Y = A_r^-1 B_r (and Z = A_r^-1 C_r when want_z), C_r kept in Cr
    void solve_layout(const OpDev& op, long ns, const long* sidx, const double* sval, long nd, const long* didx,
                      const double* dval, bool want_z) {
        reduced_system(op);
        factor();
        B.ensure(sizeof(T) * r * (ns + nd));
        Cr.ensure(sizeof(T) * r * std::max(1L, nd));
        gather(sidx, sval, ns, B.template as<T>());
        gather(didx, dval, nd, Cr.template as<T>());
        if (want_z)
            CK(cudaMemcpyAsync(B.template as<T>() + (size_t)ns * r, Cr.p, sizeof(T) * r * nd, cudaMemcpyDeviceToDevice,
                               ctx->s));
        solve(B.template as<T>(), want_z ? ns + nd : ns);
    }

    // Psi_r = C_r^T Y (n_det x n_src, rom.cpp:29-35)
    void transfer(const OpDev& op, long ns, const long* sidx, const double* sval, long nd, const long* didx,
                  const double* dval, T* Psi) {
        solve_layout(op, ns, sidx, sval, nd, didx, dval, false);
        gram<T, false>(*ctx, Cr.template as<T>(), r, nd, B.template as<T>(), r, ns, r, Psi, false, gwork);
    }

    // J[:, k] = scale * vec(sum_t w_t (V Z)[i_t,:]^T (V Y)[i_t,:])   (rom.cpp:37-67)
    void jacobian(const OpDev& op, long ns, const long* sidx, const double* sval, long nd, const long* didx,
                  const double* dval, long npar, const long* ptr, const long* sidx_k, const double* sval_k,
                  double scale, T* J) {
        Ctx& c = *ctx;
        solve_layout(op, ns, sidx, sval, nd, didx, dval, true);
        WY.ensure(sizeof(T) * n * ns);
        WZ.ensure(sizeof(T) * n * std::max(1L, nd));
        gemm<T, false>(c, V, n, r, B.template as<T>(), ns, nullptr, 0, WY.template as<T>(), n, n, false);
        gemm<T, false>(c, V, n, r, B.template as<T>() + (size_t)ns * r, nd, nullptr, 0, WZ.template as<T>(), n, n,
                       false);
        if (npar <= 0) return;
        const long nnz = ptr[npar];
        for (long k = 0; k < npar; ++k)
            if (ptr[k + 1] < ptr[k]) throw ConfigError("rom: support pointers not monotone");
        for (long t = 0; t < nnz; ++t)
            if (sidx_k[t] < 0 || sidx_k[t] >= n) throw ConfigError("rom: support index out of range");
        Pd.ensure(sizeof(long) * (npar + 1) + sizeof(long) * std::max(1L, nnz) + sizeof(double) * std::max(1L, nnz));
        long* dptr = Pd.template as<long>();
        long* didx2 = dptr + (npar + 1);
        double* dval2 = reinterpret_cast<double*>(didx2 + std::max(1L, nnz));
        CK(cudaMemcpyAsync(dptr, ptr, sizeof(long) * (npar + 1), cudaMemcpyHostToDevice, c.s));
        if (nnz > 0) {
            CK(cudaMemcpyAsync(didx2, sidx_k, sizeof(long) * nnz, cudaMemcpyHostToDevice, c.s));
            CK(cudaMemcpyAsync(dval2, sval_k, sizeof(double) * nnz, cudaMemcpyHostToDevice, c.s));
        }
        for (long k0 = 0; k0 < npar; k0 += 65535) {
            const long kk = std::min(65535L, npar - k0);
            dim3 grid((unsigned)std::max(1L, std::min<long>((ns * nd + 255) / 256, 64)), (unsigned)kk);
            rom_jacobian<T><<<grid, 256, 0, c.s>>>(WY.template as<T>(), WZ.template as<T>(), n, (int)ns, (int)nd,
                                                   dptr + k0, didx2, dval2, scale, J + (size_t)k0 * ns * nd, ns * nd);
            c.check_launch();
        }
        c.sync();
    }
};

struct RomHandle {
    int dtype = 0;
    std::unique_ptr<DevRom<double>> r;
    std::unique_ptr<DevRom<cplx>> c;
};
}  // namespace rd

struct rd_ctx {
    Ctx c;
};
struct rd_op {
    rd_ctx* ctx;
    DevOp op;
};
struct rd_basis {
    rd_ctx* ctx;
    BasisHandle h;
};

namespace {

template <class F> int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const rd::ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const rd::SolverError& e) {
        g_err = e.what();
        return 3;
    } catch (const rd::CudaError& e) {
        g_err = e.what();
        return 5;
    } catch (const rd::IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Stage a host or device buffer on the device (copy if host).
struct Staged {
    DevBuf own;
    void* p = nullptr;
    Staged(Ctx& c, const void* src, size_t bytes, int where) {
        if (where == 1 || src == nullptr) {
            p = const_cast<void*>(src);
        } else {
            own.ensure(std::max<size_t>(bytes, 16));
            CK(cudaMemcpyAsync(own.p, src, bytes, cudaMemcpyHostToDevice, c.s));
            p = own.p;
        }
    }
};
struct Out {
    Ctx& c;
    DevBuf own;
    void* dst;
    void* p;
    size_t bytes;
    int where;
    Out(Ctx& cc, void* d, size_t b, int w) : c(cc), dst(d), p(nullptr), bytes(b), where(w) {
        if (dst == nullptr) {
            p = nullptr;
        } else if (where == 1) {
            p = dst;
        } else {
            own.ensure(std::max<size_t>(bytes, 16));
            p = own.p;
        }
    }
    void finish() {
        if (dst && where == 0) {
            CK(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyDeviceToHost, c.s));
            c.sync();
        }
    }
};

size_t esize(int dtype) { return dtype == 1 ? 16 : 8; }

double gershgorin_host(const std::vector<double>& D, const std::vector<double>& mu, int d, const long* N,
                       double robin_face, double shift) {
    const long n0 = N[0], n1 = N[1], n2 = d == 3 ? N[2] : 1;
    double lm = 0.0;
    auto hm = [](double a, double b) { return 2.0 * (a * b) / (a + b); };
    for (long k = 0; k < n2; ++k)
        for (long j = 0; j < n1; ++j)
            for (long i = 0; i < n0; ++i) {
                const long p = i + n0 * (j + n1 * k);
                double diag = mu[p], off = 0.0;
                const long idx[3] = {i, j, k};
                const long len[3] = {n0, n1, n2};
                const long st[3] = {1, n0, n0 * n1};
                for (int ax = 0; ax < d; ++ax)
                    for (int dir = -1; dir <= 1; dir += 2) {
                        const long q = idx[ax] + dir;
                        if (q >= 0 && q < len[ax]) {
                            const double f = hm(D[p], D[p + dir * st[ax]]);
                            diag += f;
                            off += f;
                        } else {
                            diag += (ax == d - 1) ? robin_face : D[p];
                        }
                    }
                lm = std::max(lm, std::fabs(diag) + std::fabs(shift) + off);
            }
    return lm;
}

}  // namespace

extern "C" {

const char* rd_last_error(void) { return g_err.c_str(); }

int rd_ctx_create(int device, rd_ctx** out) {
    return guard([&] {
        auto* c = new rd_ctx();
        try {
            c->c.init(device);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}
void rd_ctx_destroy(rd_ctx* ctx) { delete ctx; }
int rd_ctx_sync(rd_ctx* ctx) {
    return guard([&] { ctx->c.sync(); });
}
int rd_ctx_mark(rd_ctx* ctx) {
    return guard([&] {
        Ctx& c = ctx->c;
        cudaEvent_t e = c.mark[c.nmark & 1];
        CK(cudaEventRecord(e, c.s));
        ++c.nmark;
    });
}
double rd_ctx_elapsed_ms(rd_ctx* ctx) {
    Ctx& c = ctx->c;
    if (c.nmark < 2) return -1.0;
    cudaEvent_t a = c.mark[(c.nmark - 2) & 1], b = c.mark[(c.nmark - 1) & 1];
    float ms = -1.f;
    if (cudaEventSynchronize(b) != cudaSuccess) return -1.0;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return -1.0;
    return ms;
}
long rd_ctx_launches(rd_ctx* ctx) { return ctx->c.launches; }

int rd_ctx_set_solver(rd_ctx* ctx, int solver) {
    return guard([&] {
        if (solver != 0 && solver != 1) throw rd::ConfigError("solver: 0 (CG / COCG) or 1 (MINRES)");
        ctx->c.solver = solver;
    });
}
int rd_ctx_get_solver(rd_ctx* ctx) { return ctx->c.solver; }
void rd_ctx_fused_check(rd_ctx* ctx, long* launches_checked, long* violations) {
    if (launches_checked) *launches_checked = ctx->c.fchk_checked;
    if (violations) *violations = ctx->c.fchk_violations;
}
void rd_ctx_profile(rd_ctx* ctx, int enable) {
    ctx->c.prof = enable != 0;
    for (auto& q : ctx->c.pc) q = Ctx::ProfClass();
}
int rd_ctx_prof_get(rd_ctx* ctx, int cls, double* ms, double* bytes, long* samples) {
    if (cls < 0 || cls >= 8) return 2;
    const auto& q = ctx->c.pc[cls];
    if (ms) *ms = q.ms;
    if (bytes) *bytes = q.bytes;
    if (samples) *samples = q.samples;
    return 0;
}
void* rd_ctx_stream(rd_ctx* ctx) { return (void*)ctx->c.s; }

int rd_op_create(rd_ctx* ctx, int d, const long* N, double robin_face, rd_op** out) {
    return guard([&] {
        if (d != 2 && d != 3) throw rd::ConfigError("operator: d must be 2 or 3");
        for (int a = 0; a < d; ++a)
            if (N[a] < 2) throw rd::ConfigError("operator: every axis needs at least 2 nodes");
        auto* o = new rd_op();
        o->ctx = ctx;
        o->op.ctx = &ctx->c;
        OpDev& od = o->op.d;
        od.d = d;
        od.N0 = (int)N[0];
        od.N1 = (int)N[1];
        od.N2 = d == 3 ? (int)N[2] : 1;
        od.n = (long)od.N0 * od.N1 * od.N2;
        od.robin_face = robin_face;
        od.shift = 0.0;
        *out = o;
    });
}
void rd_op_destroy(rd_op* op) { delete op; }

int rd_op_set_fields(rd_op* o, const double* D, const double* mu, double shift, int where) {
    return guard([&] {
        Ctx& c = o->ctx->c;
        const long n = o->op.d.n;
        o->op.D.ensure(sizeof(double) * n);
        o->op.mu.ensure(sizeof(double) * n);
        const auto kind = where == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        CK(cudaMemcpyAsync(o->op.D.p, D, sizeof(double) * n, kind, c.s));
        CK(cudaMemcpyAsync(o->op.mu.p, mu, sizeof(double) * n, kind, c.s));
        o->op.d.D = o->op.D.template as<double>();
        o->op.d.mu = o->op.mu.template as<double>();
        o->op.d.shift = shift;
        o->op.F.ensure(sizeof(double) * 4 * n);
        o->op.d.F = o->op.F.template as<double>();
        op_prepare<<<stencil_grid(o->op.d, 1), 256, 0, c.s>>>(o->op.d, o->op.F.template as<double>());
        c.check_launch();
        if (o->op.d.N0 % 2 == 0) {
            o->op.d.Fp = o->op.d.F;
            o->op.d.ldF = o->op.d.N0;
        } else {
            const long rows = (long)o->op.d.N1 * o->op.d.N2, ld = o->op.d.N0 + 1;
            o->op.Fpad.ensure(sizeof(double) * 4 * rows * ld);
            pad_fields<<<c.grid_for(4 * rows * ld, 256, 4), 256, 0, c.s>>>(o->op.d.F, n, o->op.d.N0, rows, ld,
                                                                        o->op.Fpad.template as<double>());
            c.check_launch();
            o->op.d.Fp = o->op.Fpad.template as<double>();
            o->op.d.ldF = ld;
        }
        o->op.have_fields = true;
        if (where == 0) {
            std::vector<double> Dh(D, D + n), mh(mu, mu + n);
            const long N[3] = {o->op.d.N0, o->op.d.N1, o->op.d.N2};
            o->op.lam_max = gershgorin_host(Dh, mh, o->op.d.d, N, o->op.d.robin_face, shift);
        } else {
            o->op.lam_max = 0.0;  // computed lazily by the eigensolver
        }
    });
}

double rd_op_lam_max(rd_op* op) { return op->op.lam_max; }

int rd_op_apply(rd_op* o, int dtype, const void* x, void* y, long ncols, int where) {
    return guard([&] {
        Ctx& c = o->ctx->c;
        if (!o->op.have_fields) throw rd::ConfigError("operator: fields not set");
        const long n = o->op.d.n;
        const size_t bytes = esize(dtype) * n * ncols;
        Staged xs(c, x, bytes, where);
        Out ys(c, y, bytes, where);
        if (dtype == 0)
            launch_stencil<double>(c, o->op.d, (const double*)xs.p, n, nullptr, (double*)ys.p, n, ncols);
        else
            launch_stencil<cplx>(c, o->op.d, (const cplx*)xs.p, n, nullptr, (cplx*)ys.p, n, ncols);
        ys.finish();
        if (where == 1) c.sync();
    });
}

int rd_recycled_solve(rd_op* o, int dtype, const void* U, const void* K, long c, const void* rhs, double tol,
                      long maxit, double rhs_scale, void* g, void* y, void* image, rd_report* rep, double* hist,
                      long hist_cap, int where) {
    return guard([&] {
        Ctx& cx = o->ctx->c;
        if (!o->op.have_fields) throw rd::ConfigError("operator: fields not set");
        const long n = o->op.d.n;
        const size_t es = esize(dtype);
        Staged Us(cx, c ? U : nullptr, es * n * c, where), Ks(cx, c ? K : nullptr, es * n * c, where);
        Staged rs(cx, rhs, es * n, where);
        Out gs(cx, g, es * n, where), ys(cx, y, es * n, where), is(cx, image, es * n, where);
        DevBuf gt, yt, it;
        void* gp = gs.p;
        void* yp = ys.p;
        void* ip = is.p;
        if (!gp) {
            gt.ensure(es * n);
            gp = gt.p;
        }
        if (!yp) {
            yt.ensure(es * n);
            yp = yt.p;
        }
        if (!ip) {
            it.ensure(es * n);
            ip = it.p;
        }
        SolveOut so;
        if (dtype == 0) {
            Workspace<double> ws;
            so = recycled_solve<double>(cx, o->op, (const double*)Us.p, (const double*)Ks.p, c, (const double*)rs.p, tol,
                                     maxit, rhs_scale, (double*)gp, (double*)yp, (double*)ip, ws, hist != nullptr);
        } else {
            Workspace<cplx> ws;
            so = recycled_solve<cplx>(cx, o->op, (const cplx*)Us.p, (const cplx*)Ks.p, c, (const cplx*)rs.p, tol, maxit,
                                   rhs_scale, (cplx*)gp, (cplx*)yp, (cplx*)ip, ws, hist != nullptr);
        }
        // correction norm
        double* nrm = cx.sc(3);
        if (dtype == 0)
            launch_norms<double>(cx, (const double*)gp, n, nrm);
        else
            launch_norms<cplx>(cx, (const cplx*)gp, n, nrm);
        double h;
        CK(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, cx.s));
        gs.finish();
        ys.finish();
        is.finish();
        cx.sync();
        if (rep) {
            rep->iterations = so.iterations;
            rep->converged = so.converged ? 1 : 0;
            rep->final_relres = so.final_relres;
            rep->correction_norm = std::sqrt(h);
        }
        if (hist)
            for (long i = 0; i < std::min<long>(hist_cap, (long)so.hist.size()); ++i) hist[i] = so.hist[i];
    });
}

int rd_recycle_space_from_raw(rd_ctx* ctx, int dtype, long n, long c, const void* Wr, const void* AW, void* U,
                              void* K, int where) {
    return guard([&] {
        Ctx& cx = ctx->c;
        const size_t es = esize(dtype);
        Staged Ws(cx, Wr, es * n * c, where), As(cx, AW, es * n * c, where);
        Out Us(cx, U, es * n * c, where), Ks(cx, K, es * n * c, where);
        if (dtype == 0)
            from_raw<double>(cx, n, c, (const double*)Ws.p, nullptr, (const double*)As.p, (double*)Us.p,
                             (double*)Ks.p);
        else
            from_raw<cplx>(cx, n, c, (const cplx*)Ws.p, nullptr, (const cplx*)As.p, (cplx*)Us.p, (cplx*)Ks.p);
        Us.finish();
        Ks.finish();
        cx.sync();
    });
}

int rd_initial_solutions(rd_op* o, int dtype, long nrhs, const long* bidx, const double* bval, double tol,
                         void* X0, int where, long* total_iterations) {
    return guard([&] {
        Ctx& cx = o->ctx->c;
        const long n = o->op.d.n;
        const size_t es = esize(dtype);
        if (!o->op.have_fields) throw rd::ConfigError("operator: fields not set");
        if (dtype == 0 && o->op.d.shift != 0.0) throw rd::ConfigError("real solve with a complex operator");
        Out Xs(cx, X0, es * n * nrhs, where);
        DevBuf g;
        if (!Xs.p) g.ensure(es * n * std::max(1L, nrhs));
        void* xp = Xs.p ? Xs.p : g.p;
        // batched independent solves (basis.cpp:141-149), chunked to bound the
        // 5 n-vectors per column of workspace
        const long chunk = std::max(1L, std::min(nrhs, (long)(24e9 / (5.0 * es * (double)n))));
        long tot = 0;
        if (cx.solver == 1) {
            // the reference's seed solves: MINRES column by column at 0.25 tol (basis.cpp:141-149)
            if (dtype != 0) throw rd::ConfigError("solver: MINRES (the reference's solver) is real symmetric only");
            Workspace<double> ws;
            DevBuf rhsb, yb, ib;
            rhsb.ensure(es * n);
            yb.ensure(es * n);
            ib.ensure(es * n);
            CK(cudaMemsetAsync(rhsb.p, 0, es * n, cx.s));
            const double zero = 0.0;
            for (long j = 0; j < nrhs; ++j) {
                double* rhs = rhsb.template as<double>();
                CK(cudaMemcpyAsync(rhs + bidx[j], &bval[j], sizeof(double), cudaMemcpyHostToDevice, cx.s));
                const SolveOut so = recycled_minres_dev(cx, o->op, nullptr, nullptr, 0, rhs, kInnerSafety * tol, 2 * n, 0.0,
                                                        static_cast<double*>(xp) + (size_t)j * n,
                                                        yb.template as<double>(), ib.template as<double>(), ws, false);
                CK(cudaMemcpyAsync(rhs + bidx[j], &zero, sizeof(double), cudaMemcpyHostToDevice, cx.s));
                cx.sync();
                if (!so.converged)
                    throw rd::SolverError("init_basis: MINRES failed on initial solution column " + std::to_string(j));
                tot += so.iterations;
            }
            Xs.finish();
            cx.sync();
            if (total_iterations) *total_iterations = tot;
            return;
        }
        auto run = [&](auto tag) {
            using T = decltype(tag);
            for (long j0 = 0; j0 < nrhs; j0 += chunk) {
                const long m = std::min(chunk, nrhs - j0);
                const auto st = batched_cg<T>(cx, o->op, m, bidx + j0, bval + j0, kInnerSafety * tol, 2 * n,
                                              static_cast<T*>(xp) + (size_t)j0 * n);
                for (long j = 0; j < m; ++j) {
                    if (!st[j].converged)
                        throw rd::SolverError("init_basis: CG failed on initial solution column " +
                                              std::to_string(j0 + j));
                    tot += st[j].it;
                    VLOG(2, "X0 column %ld: %d its", j0 + j, st[j].it);
                }
            }
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
        Xs.finish();
        cx.sync();
        if (total_iterations) *total_iterations = tot;
    });
}

// fom_transfer (rom.cpp:86-91) with the batched CG / COCG in place of MINRES
int rd_fom_transfer(rd_op* o, int dtype, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, double tol, void* Psi, int where,
                    long* total_iterations) {
    return guard([&] {
        Ctx& cx = o->ctx->c;
        const long n = o->op.d.n;
        const size_t es = esize(dtype);
        if (!o->op.have_fields) throw rd::ConfigError("operator: fields not set");
        if (dtype == 0 && o->op.d.shift != 0.0) throw rd::ConfigError("real solve with a complex operator");
        if (n_src <= 0 || n_det <= 0) throw rd::ConfigError("fom: need sources and detectors");
        for (long d = 0; d < n_det; ++d)
            if (det_idx[d] < 0 || det_idx[d] >= n) throw rd::ConfigError("fom: detector index out of range");
        Out ps(cx, Psi, es * n_src * n_det, where);
        DevBuf Xb, ix, vx;
        Xb.ensure(es * n * n_src);
        ix.ensure(sizeof(long) * n_det);
        vx.ensure(sizeof(double) * n_det);
        long tot = 0;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const auto st = batched_cg<T>(cx, o->op, n_src, src_idx, src_val, tol, 2 * n, Xb.template as<T>());
            for (long j = 0; j < n_src; ++j) {
                if (!st[j].converged) throw rd::SolverError("fom: CG did not converge");
                tot += st[j].it;
            }
            CK(cudaMemcpyAsync(ix.p, det_idx, sizeof(long) * n_det, cudaMemcpyHostToDevice, cx.s));
            CK(cudaMemcpyAsync(vx.p, det_val, sizeof(double) * n_det, cudaMemcpyHostToDevice, cx.s));
            fom_gather<T><<<(int)((n_src * n_det + 255) / 256), 256, 0, cx.s>>>(
                Xb.template as<T>(), n, (int)n_src, ix.template as<long>(), vx.template as<double>(), (int)n_det,
                static_cast<T*>(ps.p));
            cx.check_launch();
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
        ps.finish();
        cx.sync();
        if (total_iterations) *total_iterations = tot;
    });
}

// fom_jacobian / jacobian_from_solutions (rom.cpp:101-129): X = A^-1 B~,
// Z = A^-1 C~ by one batched solve, then the support-row contraction of the
// reduced model's kernel with Wy = X, Wz = Z.
int rd_fom_jacobian(rd_op* o, int dtype, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, long n_par, const long* sup_ptr, const long* sup_idx,
                    const double* sup_val, double scale, double tol, void* J, int where) {
    return guard([&] {
        Ctx& cx = o->ctx->c;
        const long n = o->op.d.n;
        const size_t es = esize(dtype);
        if (!o->op.have_fields) throw rd::ConfigError("operator: fields not set");
        if (dtype == 0 && o->op.d.shift != 0.0) throw rd::ConfigError("real solve with a complex operator");
        if (n_src <= 0 || n_det <= 0) throw rd::ConfigError("fom: need sources and detectors");
        if (n_par < 0 || (n_par > 0 && !sup_ptr)) throw rd::ConfigError("fom: bad parameter supports");
        const long nnz = n_par > 0 ? sup_ptr[n_par] : 0;
        for (long k = 0; k < n_par; ++k)
            if (sup_ptr[k + 1] < sup_ptr[k]) throw rd::ConfigError("fom: support pointers not monotone");
        for (long t = 0; t < nnz; ++t)
            if (sup_idx[t] < 0 || sup_idx[t] >= n) throw rd::ConfigError("fom: support index out of range");
        Out js(cx, J, es * n_src * n_det * std::max(1L, n_par), where);
        const long m = n_src + n_det;
        std::vector<long> bi(m);
        std::vector<double> bv(m);
        for (long j = 0; j < n_src; ++j) bi[j] = src_idx[j], bv[j] = src_val[j];
        for (long j = 0; j < n_det; ++j) bi[n_src + j] = det_idx[j], bv[n_src + j] = det_val[j];
        DevBuf Xb, Pd;
        Xb.ensure(es * n * m);
        Pd.ensure(sizeof(long) * (n_par + 1) + sizeof(long) * std::max(1L, nnz) + sizeof(double) * std::max(1L, nnz));
        long* dptr = Pd.template as<long>();
        long* didx = dptr + (n_par + 1);
        double* dval = reinterpret_cast<double*>(didx + std::max(1L, nnz));
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const auto st = batched_cg<T>(cx, o->op, m, bi.data(), bv.data(), tol, 2 * n, Xb.template as<T>());
            for (long j = 0; j < m; ++j)
                if (!st[j].converged) throw rd::SolverError("fom: CG did not converge");
            if (n_par <= 0) return;
            CK(cudaMemcpyAsync(dptr, sup_ptr, sizeof(long) * (n_par + 1), cudaMemcpyHostToDevice, cx.s));
            if (nnz > 0) {
                CK(cudaMemcpyAsync(didx, sup_idx, sizeof(long) * nnz, cudaMemcpyHostToDevice, cx.s));
                CK(cudaMemcpyAsync(dval, sup_val, sizeof(double) * nnz, cudaMemcpyHostToDevice, cx.s));
            }
            const T* X = Xb.template as<T>();
            for (long k0 = 0; k0 < n_par; k0 += 65535) {
                const long kk = std::min(65535L, n_par - k0);
                dim3 grid((unsigned)std::max(1L, std::min<long>((n_src * n_det + 255) / 256, 64)), (unsigned)kk);
                rom_jacobian<T><<<grid, 256, 0, cx.s>>>(X, X + (size_t)n_src * n, n, (int)n_src, (int)n_det, dptr + k0,
                                                        didx, dval, scale,
                                                        static_cast<T*>(js.p) + (size_t)k0 * n_src * n_det,
                                                        n_src * n_det);
                cx.check_launch();
            }
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
        js.finish();
        cx.sync();
    });
}

int rd_basis_create(rd_ctx* ctx, int dtype, long n, long ku, long nrhs, const void* U0, const void* X0, long cap,
                    int where, rd_basis** out) {
    return guard([&] {
        Ctx& cx = ctx->c;
        auto* b = new rd_basis();
        b->ctx = ctx;
        b->h.ctx = &cx;
        b->h.dtype = dtype;
        auto setup = [&](auto& gb, auto tag) {
            using T = decltype(tag);
            gb.reset(new DevBasis<T>());
            DevBasis<T>& B = *gb;
            B.ctx = &cx;
            B.n = n;
            B.cap = cap;
            B.ku = ku;
            B.reserve(std::max(ku + nrhs, 16L));
            const auto kind = where == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
            if (ku) CK(cudaMemcpyAsync(B.Vp(), U0, sizeof(T) * n * ku, kind, cx.s));
            if (nrhs) CK(cudaMemcpyAsync(B.Vp() + (size_t)n * ku, X0, sizeof(T) * n * nrhs, kind, cx.s));
            B.cols = ku + nrhs;
            B.markers.assign(ku, kColEigenvector);
            B.markers.insert(B.markers.end(), nrhs, kColInitialSolution);
            B.spaces.assign(nrhs, {});
            for (long j = 0; j < nrhs; ++j) {
                for (long i = 0; i < ku; ++i) B.spaces[j].push_back((int)i);
                B.spaces[j].push_back((int)(ku + j));
            }
            cx.sync();
        };
        if (dtype == 0)
            setup(b->h.r, double{});
        else
            setup(b->h.c, cplx{});
        *out = b;
    });
}
void rd_basis_destroy(rd_basis* b) { delete b; }

#define BASIS_DISPATCH(b, ...)     \
    if ((b)->h.dtype == 0) {       \
        auto& B = *(b)->h.r;       \
        __VA_ARGS__;               \
    } else {                       \
        auto& B = *(b)->h.c;       \
        __VA_ARGS__;               \
    }

long rd_basis_cols(rd_basis* b) {
    long v = 0;
    BASIS_DISPATCH(b, v = B.cols);
    return v;
}
int rd_basis_factored(rd_basis* b) {
    int v = 0;
    BASIS_DISPATCH(b, v = B.factored ? 1 : 0);
    return v;
}
long rd_basis_eig_block(rd_basis* b) {
    long v = 0;
    BASIS_DISPATCH(b, v = B.ku);
    return v;
}
long rd_basis_batched_solves(rd_basis* b) {
    long v = 0;
    BASIS_DISPATCH(b, v = B.stats_batched_rhs);
    return v;
}
void* rd_basis_device_ptr(rd_basis* b, int which) {
    void* p = nullptr;
    const int rc = guard([&] {
        BASIS_DISPATCH(b, {
            if (which >= 2) {
                if (!B.factored || !B.Wm.p) throw ConfigError("basis has no W = V R^-1 (refresh first)");
                B.materialize_W();
            }
            p = which == 0 ? (void*)B.Vp() : which == 1 ? (void*)B.Kp() : (void*)B.Wp();
        });
    });
    return rc == 0 ? p : nullptr;
}
int rd_basis_set_rhs_hook(rd_basis* b, int (*fn)(void*, int, long), void* user) {
    return guard([&] {
        BASIS_DISPATCH(b, {
            B.hook = fn;
            B.hook_user = user;
        });
    });
}
int rd_basis_get(rd_basis* b, int which, void* out) {
    return guard([&] {
        BASIS_DISPATCH(b, {
            using T = std::remove_reference_t<decltype(B.R[0])>;
            if (which != 0 && !B.factored) throw ConfigError("basis has no image factor yet (refresh first)");
            if (which == 2) {
                T* o = (T*)out;
                for (long j = 0; j < B.cols; ++j)
                    for (long i = 0; i < B.cols; ++i) o[i + j * B.cols] = i <= j ? B.Rat(i, j) : Sc<T>::zero();
            } else {
                if (which == 3) B.materialize_W();
                const T* src = which == 0 ? B.Vp() : which == 1 ? B.Kp() : B.Wp();
                CK(cudaMemcpyAsync(out, src, sizeof(T) * B.n * B.cols, cudaMemcpyDeviceToHost, b->ctx->c.s));
                b->ctx->c.sync();
            }
        });
    });
}
int rd_basis_markers(rd_basis* b, uint8_t* out) {
    return guard([&] { BASIS_DISPATCH(b, std::memcpy(out, B.markers.data(), B.markers.size())); });
}
long rd_basis_space(rd_basis* b, long j, int* out) {
    long m = -1;
    BASIS_DISPATCH(b, {
        if (j >= 0 && j < (long)B.spaces.size()) {
            m = (long)B.spaces[j].size();
            if (out) std::memcpy(out, B.spaces[j].data(), sizeof(int) * m);
        }
    });
    return m;
}
int rd_basis_refresh(rd_basis* b, rd_op* op) {
    return guard([&] {
        BASIS_DISPATCH(b, {
            if (B.raw_only) throw rd::ConfigError("refresh: handle is a per-RHS recycler");
            B.refresh(op->op);
        });
    });
}
int rd_basis_append(rd_basis* b, const void* y, const void* z, int marker, int where, int* appended) {
    return guard([&] {
        Ctx& cx = b->ctx->c;
        BASIS_DISPATCH(b, {
            if (B.raw_only) throw rd::ConfigError("append: handle is a per-RHS recycler");
            using T = std::remove_reference_t<decltype(B.R[0])>;
            Staged ys(cx, y, sizeof(T) * B.n, where), zs(cx, z, sizeof(T) * B.n, where);
            const bool ok = B.append((const T*)ys.p, (const T*)zs.p, (uint8_t)marker);
            if (appended) *appended = ok ? 1 : 0;
        });
    });
}
int rd_basis_solve_projected(rd_basis* b, const void* rhs, void* x, void* coords, int where) {
    return guard([&] {
        Ctx& cx = b->ctx->c;
        BASIS_DISPATCH(b, {
            using T = std::remove_reference_t<decltype(B.R[0])>;
            constexpr int W = Sc<T>::W;
            const long n = B.n, r = B.cols;
            Staged bs(cx, rhs, sizeof(T) * n, where);
            Out xs(cx, x, sizeof(T) * n, where);
            DevBuf w, zero, xt;
            w.ensure(sizeof(double) * W * std::max(1L, r));
            zero.ensure(sizeof(T) * n);
            CK(cudaMemsetAsync(zero.p, 0, sizeof(T) * n, cx.s));
            ts_T_launch<T, true>(cx, B.Kp(), n, r, (const T*)bs.p, n, w.template as<double>());
            void* xp = xs.p;
            if (!xp) {
                xt.ensure(sizeof(T) * n);
                xp = xt.p;
            }
            B.materialize_W();
            ts_N_launch<T>(cx, B.Wp(), n, r, zero.template as<T>(), (T*)xp, n, w.template as<double>(), -1.0);
            xs.finish();
            if (coords) {
                // c = R^-1 w (host triangular solve on the r x r factor)
                std::vector<T> wc(r);
                CK(cudaMemcpyAsync(wc.data(), w.p, sizeof(T) * r, cudaMemcpyDeviceToHost, cx.s));
                cx.sync();
                for (long i = r - 1; i >= 0; --i) {
                    T s = wc[i];
                    for (long k = i + 1; k < r; ++k) s = Sc<T>::sub(s, Sc<T>::mul(B.Rat(i, k), wc[k]));
                    wc[i] = Sc<T>::div(s, B.Rat(i, i));
                }
                std::memcpy(coords, wc.data(), sizeof(T) * r);
            }
            cx.sync();
        });
    });
}

int rd_process_system(rd_basis* b, rd_op* op, long nrhs, const long* bidx, const double* bval, double tol,
                      int system_index, long maxit, void* X, int where, double* log, long* inner_iterations,
                      long* appends) {
    return guard([&] {
        Ctx& cx = b->ctx->c;
        if (!op->op.have_fields) throw rd::ConfigError("operator: fields not set");
        BASIS_DISPATCH(b, {
            using T = std::remove_reference_t<decltype(B.R[0])>;
            if (B.n != op->op.d.n) throw rd::ConfigError("process_system: dimension mismatch");
            if (B.raw_only) throw rd::ConfigError("process_system: handle is a per-RHS recycler");
            Out xs(cx, X, sizeof(T) * B.n * nrhs, where);
            if (X && where == 0) B.X.ensure(sizeof(T) * B.n * nrhs);
            T* Xd = X ? (where == 0 ? B.X.template as<T>() : (T*)X) : nullptr;
            std::vector<LogRow> lg;
            long its = 0, app = 0;
            process_system<T>(B, op->op, nrhs, bidx, bval, tol, system_index, maxit, Xd, lg, its, app);
            if (X && where == 0) {
                CK(cudaMemcpyAsync(X, Xd, sizeof(T) * B.n * nrhs, cudaMemcpyDeviceToHost, cx.s));
                cx.sync();
            }
            if (log)
                for (size_t t = 0; t < lg.size(); ++t) {
                    log[5 * t + 0] = lg[t].system;
                    log[5 * t + 1] = lg[t].rhs;
                    log[5 * t + 2] = lg[t].init_relres;
                    log[5 * t + 3] = lg[t].iterations;
                    log[5 * t + 4] = lg[t].appended ? 1.0 : 0.0;
                }
            if (inner_iterations) *inner_iterations = its;
            if (appends) *appends = app;
        });
    });
}

int rd_per_rhs_create(rd_ctx* ctx, int dtype, long n, long ku, long nrhs, const void* U0, const void* X0, int where,
                      rd_basis** out) {
    const int rc = rd_basis_create(ctx, dtype, n, ku, nrhs, U0, X0, 0, where, out);
    if (rc == 0) BASIS_DISPATCH(*out, B.raw_only = true);
    return rc;
}

int rd_per_rhs_solve_system(rd_basis* b, rd_op* op, long nrhs, const long* bidx, const double* bval, double tol,
                            int system_index, long maxit, void* X, int where, double* log, long* inner_iterations,
                            long* appends) {
    return guard([&] {
        Ctx& cx = b->ctx->c;
        if (!op->op.have_fields) throw rd::ConfigError("operator: fields not set");
        BASIS_DISPATCH(b, {
            using T = std::remove_reference_t<decltype(B.R[0])>;
            if (!B.raw_only) throw rd::ConfigError("per-RHS recycler: handle is a global basis (rd_per_rhs_create)");
            if (B.n != op->op.d.n) throw rd::ConfigError("per-RHS recycler: dimension mismatch");
            Out xs(cx, X, sizeof(T) * B.n * nrhs, where);
            if (X && where == 0) B.X.ensure(sizeof(T) * B.n * nrhs);
            T* Xd = X ? (where == 0 ? B.X.template as<T>() : (T*)X) : nullptr;
            std::vector<LogRow> lg;
            long its = 0, app = 0;
            per_rhs_solve_system<T>(B, op->op, nrhs, bidx, bval, tol, system_index, maxit, Xd, lg, its, app);
            if (X && where == 0) {
                CK(cudaMemcpyAsync(X, Xd, sizeof(T) * B.n * nrhs, cudaMemcpyDeviceToHost, cx.s));
                cx.sync();
            }
            if (log)
                for (size_t t = 0; t < lg.size(); ++t) {
                    log[5 * t + 0] = lg[t].system;
                    log[5 * t + 1] = lg[t].rhs;
                    log[5 * t + 2] = lg[t].init_relres;
                    log[5 * t + 3] = lg[t].iterations;
                    log[5 * t + 4] = lg[t].appended ? 1.0 : 0.0;
                }
            if (inner_iterations) *inner_iterations = its;
            if (appends) *appends = app;
        });
    });
}

int rd_smallest_eigenpairs(rd_op* op, long k, double tol, double* lambda, void* U, int where) {
    return guard([&] {
        Ctx& cx = op->ctx->c;
        if (!op->op.have_fields) throw rd::ConfigError("operator: fields not set");
        const long n = op->op.d.n;
        Out Us(cx, U, sizeof(double) * n * k, where);
        DevBuf tmp;
        void* up = Us.p;
        if (!up) {
            tmp.ensure(sizeof(double) * n * k);
            up = tmp.p;
        }
        std::vector<double> lam;
        // the seed is defined on the omega = 0 (real SPD) operator
        const double sh = op->op.d.shift;
        op->op.d.shift = 0.0;
        try {
            smallest_eigenpairs_dev(cx, op->op, k, tol, lam, (double*)up);
        } catch (...) {
            op->op.d.shift = sh;
            throw;
        }
        op->op.d.shift = sh;
        Us.finish();
        if (lambda)
            for (long i = 0; i < k; ++i) lambda[i] = lam[i];
    });
}

int rd_rrqr(rd_ctx* ctx, int dtype, long n, long m, const void* A, double tol, int normalize, long* rank, long* perm,
            double* rdiag, void* Q, int where) {
    return guard([&] {
        Ctx& cx = ctx->c;
        const size_t es = esize(dtype);
        Staged As(cx, A, es * n * m, where);
        std::vector<long> pv;
        std::vector<double> rd_;
        DevBuf Qd;
        long rk = 0;
        if (dtype == 0)
            rk = rrqr_dev<double>(cx, n, m, (const double*)As.p, tol, normalize != 0, pv, rd_, Qd);
        else
            rk = rrqr_dev<cplx>(cx, n, m, (const cplx*)As.p, tol, normalize != 0, pv, rd_, Qd);
        *rank = rk;
        for (long j = 0; j < m; ++j) perm[j] = pv[j];
        for (long j = 0; j < m; ++j) rdiag[j] = j < (long)rd_.size() ? rd_[j] : 0.0;
        if (Q && rk > 0) {
            const auto kind = where == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
            CK(cudaMemcpyAsync(Q, Qd.p, es * n * rk, kind, cx.s));
        }
        cx.sync();
    });
}


// ---------------------------------------------------------- bench hooks ---
// Kernel-level timing hooks for the C5 sweep (scripts/sweep.py): run each
// recycle-space projection kernel `iters` times on an n x c basis of seeded
// random values and return the mean device time per launch (CUDA events).
int rd_bench_projection(rd_ctx* ctx, int dtype, long n, long c, int iters, double* ms_out) {
    return guard([&] {
        Ctx& cx = ctx->c;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const long npad = padded_rows(n);
            DevBuf K, x, r, p, s, y;
            K.ensure(sizeof(T) * npad * c);
            for (DevBuf* b : {&x, &r, &p, &s, &y}) {
                b->ensure(sizeof(T) * npad);
                CK(cudaMemsetAsync(b->p, 0, b->bytes, cx.s));
            }
            vec_randn<<<cx.grid_for(npad * c * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(K.template as<double>(),
                                                                                 npad * c * Sc<T>::W, 7);
            vec_randn<<<cx.grid_for(n * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(x.template as<double>(), n * Sc<T>::W, 8);
            cx.check_launch();
            CGState init{};
            init.maxit = 1 << 30;
            init.tol = 0.0;
            init.scale = 1.0;
            CGState* st = cx.cgst.template as<CGState>();
            cx.st_host[0] = init;
            CK(cudaMemcpyAsync(st, &cx.st_host[0], sizeof(CGState), cudaMemcpyHostToDevice, cx.s));
            double* c1 = cx.sc(1);
            double* c2 = cx.sc(2);
            CK(cudaMemsetAsync(c1, 0, sizeof(double) * 8192 * 2, cx.s));
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            for (int mode = 0; mode < 3; ++mode) {
                auto launch = [&]() {
                    if (mode == 0)
                        ts_tma_launch<T, 0>(cx, K.template as<T>(), (int)c, n, x.template as<T>(), nullptr, nullptr, c1);
                    else if (mode == 1)
                        ts_tma_launch<T, 1>(cx, K.template as<T>(), (int)c, n, x.template as<T>(), y.template as<T>(),
                                            c1, c2);
                    else
                        ts_tma_launch<T, 2>(cx, K.template as<T>(), (int)c, n, x.template as<T>(), nullptr, c2,
                                            nullptr, r.template as<T>(), p.template as<T>(), s.template as<T>(),
                                            y.template as<T>(), st);
                };
                for (int w = 0; w < 3; ++w) launch();
                CK(cudaEventRecord(a, cx.s));
                for (int t = 0; t < iters; ++t) launch();
                CK(cudaEventRecord(b, cx.s));
                CK(cudaEventSynchronize(b));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, a, b));
                ms_out[mode] = ms / iters;
            }
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
    });
}

// Gram G = X^T X (sym != 0, upper tiles + mirror) or X^T Y timing on seeded
// random n x a / n x b blocks: mean device ms per call.
int rd_bench_gram(rd_ctx* ctx, int dtype, long n, long a, long b, int sym, int iters, double* ms_out) {
    return guard([&] {
        Ctx& cx = ctx->c;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            DevBuf x, y, g, work;
            x.ensure(sizeof(T) * n * a);
            y.ensure(sizeof(T) * n * b);
            g.ensure(sizeof(T) * a * b);
            vec_randn<<<cx.grid_for(n * a * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(x.template as<double>(),
                                                                               n * a * Sc<T>::W, 11);
            vec_randn<<<cx.grid_for(n * b * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(y.template as<double>(),
                                                                               n * b * Sc<T>::W, 12);
            cx.check_launch();
            const T* Y = sym ? x.template as<T>() : y.template as<T>();
            const long bb = sym ? a : b;
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            for (int w = 0; w < 2; ++w)
                gram<T, false>(cx, x.template as<T>(), n, a, Y, n, bb, n, g.template as<T>(), sym != 0, work);
            CK(cudaEventRecord(e0, cx.s));
            for (int t = 0; t < iters; ++t)
                gram<T, false>(cx, x.template as<T>(), n, a, Y, n, bb, n, g.template as<T>(), sym != 0, work);
            CK(cudaEventRecord(e1, cx.s));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            *ms_out = ms / iters;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
    });
}

// Mean device ms of the tall GEMM Z = X M (n x a times a x b, the refresh's
// K = Y S^-1 / W S^-1 products; upper = M upper triangular) on seeded data.
int rd_bench_gemm(rd_ctx* ctx, int dtype, long n, long a, long b, int upper, int iters, double* ms_out) {
    return guard([&] {
        Ctx& cx = ctx->c;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            DevBuf x, m, z;
            x.ensure(sizeof(T) * n * a);
            m.ensure(sizeof(T) * a * b);
            z.ensure(sizeof(T) * n * b);
            vec_randn<<<cx.grid_for(n * a * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(x.template as<double>(),
                                                                               n * a * Sc<T>::W, 21);
            vec_randn<<<cx.grid_for(a * b * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(m.template as<double>(),
                                                                               a * b * Sc<T>::W, 22);
            cx.check_launch();
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            for (int w = 0; w < 2; ++w)
                gemm<T, false>(cx, x.template as<T>(), n, a, m.template as<T>(), b, nullptr, 0, z.template as<T>(), n,
                               n, upper != 0);
            CK(cudaEventRecord(e0, cx.s));
            for (int t = 0; t < iters; ++t)
                gemm<T, false>(cx, x.template as<T>(), n, a, m.template as<T>(), b, nullptr, 0, z.template as<T>(), n,
                               n, upper != 0);
            CK(cudaEventRecord(e1, cx.s));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            *ms_out = ms / iters;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
    });
}

// Multi-column stencil apply timing on the operator's current fields.
int rd_bench_stencil(rd_op* o, int dtype, long ncols, int iters, double* ms_out) {
    return guard([&] {
        Ctx& cx = o->ctx->c;
        const long n = o->op.d.n;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            DevBuf x, y;
            x.ensure(sizeof(T) * n * ncols);
            y.ensure(sizeof(T) * n * ncols);
            vec_randn<<<cx.grid_for(n * ncols * Sc<T>::W, 256, 8), 256, 0, cx.s>>>(x.template as<double>(),
                                                                                   n * ncols * Sc<T>::W, 9);
            cx.check_launch();
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            for (int w = 0; w < 3; ++w)
                launch_stencil<T>(cx, o->op.d, x.template as<T>(), n, nullptr, y.template as<T>(), n, ncols);
            CK(cudaEventRecord(a, cx.s));
            for (int t = 0; t < iters; ++t)
                launch_stencil<T>(cx, o->op.d, x.template as<T>(), n, nullptr, y.template as<T>(), n, ncols);
            CK(cudaEventRecord(b, cx.s));
            CK(cudaEventSynchronize(b));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, a, b));
            *ms_out = ms / iters;
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
    });
}


// Explicit residual check of a solution block (test_basis.cpp:180-193 at any
// size): out[j] = ||b_j - A x_j|| / ||b_j|| with b_j = bval[j] e_{bidx[j]}.
int rd_residual_norms(rd_op* o, int dtype, long nrhs, const long* bidx, const double* bval, const void* X, int where,
                      double* out) {
    return guard([&] {
        Ctx& cx = o->ctx->c;
        const long n = o->op.d.n;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Staged Xs(cx, X, sizeof(T) * n * nrhs, where);
            DevBuf AX, idxd, vald;
            const long chunk = 16;
            AX.ensure(sizeof(T) * n * chunk);
            idxd.ensure(sizeof(long) * nrhs);
            vald.ensure(sizeof(double) * nrhs);
            std::vector<double> negval(bval, bval + nrhs);
            for (auto& v : negval) v = -v;
            CK(cudaMemcpyAsync(idxd.p, bidx, sizeof(long) * nrhs, cudaMemcpyHostToDevice, cx.s));
            CK(cudaMemcpyAsync(vald.p, negval.data(), sizeof(double) * nrhs, cudaMemcpyHostToDevice, cx.s));
            for (long j0 = 0; j0 < nrhs; j0 += chunk) {
                const long cc = std::min(chunk, nrhs - j0);
                launch_stencil<T>(cx, o->op.d, (const T*)Xs.p + (size_t)j0 * n, n, nullptr, AX.template as<T>(), n, cc);
                // A x_j - b_j
                scatter_add_rhs<T><<<1, 128, 0, cx.s>>>(AX.template as<T>(), n, idxd.template as<long>() + j0,
                                                       vald.template as<double>() + j0, (int)cc);
                cx.check_launch();
                for (long t = 0; t < cc; ++t) {
                    double* nrm = cx.sc(3);
                    launch_norms<T>(cx, AX.template as<T>() + (size_t)t * n, n, nrm);
                    double h;
                    CK(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, cx.s));
                    cx.sync();
                    out[j0 + t] = std::sqrt(h) / std::fabs(bval[j0 + t]);
                }
            }
        };
        if (dtype == 0)
            run(double{});
        else
            run(cplx{});
    });
}


// Algorithm 1 compression of a finished build (acceptance.cpp:368-383, BASELINE
// RRQR): releases the factorisation workspace (W, K_img, scratch), runs the
// RRQR directly on V's buffer and leaves the orthonormal compressed basis Q
// (n x rank) as the basis' V. The basis is final afterwards (no more
// refresh / process_system).
int rd_basis_compress(rd_basis* b, double tol, int normalize, long* rank, long* perm, double* rdiag) {
    return guard([&] {
        Ctx& cx = b->ctx->c;
        BASIS_DISPATCH(b, {
            using T = std::remove_reference_t<decltype(B.R[0])>;
            const long n = B.n, m = B.cols;
            B.Wm.~DevBuf();
            new (&B.Wm) DevBuf();
            B.K.~DevBuf();
            new (&B.K) DevBuf();
            B.Ktmp.~DevBuf();
            new (&B.Ktmp) DevBuf();
            B.AW.~DevBuf();
            new (&B.AW) DevBuf();
            std::vector<long> pv;
            std::vector<double> rd_;
            DevBuf Q;
            const long rk = rrqr_dev<T>(cx, n, m, B.Vp(), tol, normalize != 0, pv, rd_, Q, B.Vp());
            if (rk > 0) CK(cudaMemcpyAsync(B.Vp(), Q.p, sizeof(T) * n * rk, cudaMemcpyDeviceToDevice, cx.s));
            cx.sync();
            B.cols = rk;
            B.factored = false;
            B.wvalid = 0;  // W (freed above) must be re-formed after a new refresh
            B.markers.assign(rk, kColCorrection);
            *rank = rk;
            for (long j = 0; j < m; ++j) perm[j] = pv[j];
            for (long j = 0; j < m; ++j) rdiag[j] = j < (long)rd_.size() ? rd_[j] : 0.0;
        });
    });
}

struct rd_rom {
    rd_ctx* ctx;
    rd::RomHandle h;
};

#define ROM_DISPATCH(rm, ...)        \
    if ((rm)->h.dtype == 0) {        \
        auto& M = *(rm)->h.r;        \
        __VA_ARGS__;                 \
    } else {                         \
        auto& M = *(rm)->h.c;        \
        __VA_ARGS__;                 \
    }

static void rom_check_op(rd_rom* rm, rd_op* op) {
    if (!op->op.have_fields) throw rd::ConfigError("operator: fields not set");
    if (rm->h.dtype == 0 && op->op.d.shift != 0.0)
        throw rd::ConfigError("rom: real reduced model with a complex (omega != 0) operator");
}

int rd_rom_create(rd_ctx* ctx, int dtype, long n, long r, const void* V, int where, rd_rom** out) {
    return guard([&] {
        if (dtype != 0 && dtype != 1) throw rd::ConfigError("rom: dtype must be 0 (f64) or 1 (c128)");
        if (!V) throw rd::ConfigError("rom: V is null");
        auto rm = std::make_unique<rd_rom>();
        rm->ctx = ctx;
        rm->h.dtype = dtype;
        if (dtype == 0) {
            rm->h.r = std::make_unique<rd::DevRom<double>>();
            rm->h.r->init(ctx->c, n, r, V, where);
        } else {
            rm->h.c = std::make_unique<rd::DevRom<cplx>>();
            rm->h.c->init(ctx->c, n, r, V, where);
        }
        *out = rm.release();
    });
}

void rd_rom_destroy(rd_rom* rm) { delete rm; }

long rd_rom_order(rd_rom* rm) {
    long v = 0;
    ROM_DISPATCH(rm, v = M.r);
    return v;
}

int rd_rom_E(rd_rom* rm, void* E, int where) {
    return guard([&] {
        ROM_DISPATCH(rm, {
            using T = std::remove_const_t<std::remove_pointer_t<decltype(M.V)>>;
            Out es(rm->ctx->c, E, sizeof(T) * M.r * M.r, where);
            CK(cudaMemcpyAsync(es.p, M.E.p, sizeof(T) * M.r * M.r, cudaMemcpyDeviceToDevice, rm->ctx->c.s));
            es.finish();
            if (where == 1) rm->ctx->c.sync();
        });
    });
}

int rd_rom_reduced_system(rd_rom* rm, rd_op* op, void* Ar, int where) {
    return guard([&] {
        rom_check_op(rm, op);
        ROM_DISPATCH(rm, {
            using T = std::remove_const_t<std::remove_pointer_t<decltype(M.V)>>;
            M.reduced_system(op->op.d);
            Out as(rm->ctx->c, Ar, sizeof(T) * M.r * M.r, where);
            CK(cudaMemcpyAsync(as.p, M.Ar.p, sizeof(T) * M.r * M.r, cudaMemcpyDeviceToDevice, rm->ctx->c.s));
            as.finish();
            if (where == 1) rm->ctx->c.sync();
        });
    });
}

int rd_rom_transfer(rd_rom* rm, rd_op* op, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, void* Psi, int where) {
    return guard([&] {
        rom_check_op(rm, op);
        if (n_src <= 0 || n_det <= 0) throw rd::ConfigError("rom: need sources and detectors");
        ROM_DISPATCH(rm, {
            using T = std::remove_const_t<std::remove_pointer_t<decltype(M.V)>>;
            Out ps(rm->ctx->c, Psi, sizeof(T) * n_det * n_src, where);
            M.transfer(op->op.d, n_src, src_idx, src_val, n_det, det_idx, det_val, static_cast<T*>(ps.p));
            ps.finish();
            if (where == 1) rm->ctx->c.sync();
        });
    });
}

int rd_rom_jacobian(rd_rom* rm, rd_op* op, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, long n_par, const long* sup_ptr, const long* sup_idx,
                    const double* sup_val, double scale, void* J, int where) {
    return guard([&] {
        rom_check_op(rm, op);
        if (n_src <= 0 || n_det <= 0) throw rd::ConfigError("rom: need sources and detectors");
        if (n_par < 0 || (n_par > 0 && !sup_ptr)) throw rd::ConfigError("rom: bad parameter supports");
        ROM_DISPATCH(rm, {
            using T = std::remove_const_t<std::remove_pointer_t<decltype(M.V)>>;
            Out js(rm->ctx->c, J, sizeof(T) * n_src * n_det * std::max(1L, n_par), where);
            M.jacobian(op->op.d, n_src, src_idx, src_val, n_det, det_idx, det_val, n_par, sup_ptr, sup_idx, sup_val,
                       scale, static_cast<T*>(js.p));
            js.finish();
            if (where == 1) rm->ctx->c.sync();
        });
    });
}

// ------------------------------------------------------------------ ROMB ---
// Basis file (src/io.cpp:77-110): "ROMB", u32 version, u64 n, u64 r, the
// column-major data, r marker bytes, host little-endian. Version 1 is the
// reference's f64 layout, written bit-exactly; version 2 (complex bases)
// inserts one dtype byte (0 f64, 1 c128) after r.
namespace {
struct RombHeader {
    uint32_t version = 0;
    uint64_t n = 0, r = 0;
    int dtype = 0;
    long data_off = 0;
};

RombHeader romb_header(std::FILE* f, const std::string& path) {
    char magic[4];
    RombHeader h;
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "ROMB", 4) != 0)
        throw rd::IoError(path + ": not a basis file");
    if (std::fread(&h.version, 4, 1, f) != 1) throw rd::IoError(path + ": truncated basis file");
    if (h.version != 1 && h.version != 2) throw rd::IoError(path + ": unsupported basis file version");
    if (std::fread(&h.n, 8, 1, f) != 1 || std::fread(&h.r, 8, 1, f) != 1)
        throw rd::IoError(path + ": truncated basis file");
    if (h.version == 2) {
        uint8_t dt = 0;
        if (std::fread(&dt, 1, 1, f) != 1) throw rd::IoError(path + ": truncated basis file");
        if (dt > 1) throw rd::IoError(path + ": unknown dtype in basis file");
        h.dtype = dt;
    }
    h.data_off = std::ftell(f);
    return h;
}

struct File {
    std::FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};
constexpr size_t kRombChunk = size_t(1) << 28;  // device <-> host staging, 256 MB
}  // namespace

int rd_romb_write(const char* path, int dtype, long n, long r, const void* V, const uint8_t* markers, int where,
                  rd_ctx* ctx) {
    return guard([&] {
        if (dtype != 0 && dtype != 1) throw rd::ConfigError("romb: dtype must be 0 (f64) or 1 (c128)");
        if (!markers && r > 0) throw rd::IoError("basis file: marker count must equal column count");
        if (n < 0 || r < 0) throw rd::ConfigError("romb: negative dimensions");
        if (where == 1 && !ctx) throw rd::ConfigError("romb: a context is needed for device data");
        File out(path, "wb");
        if (!out.f) throw rd::IoError(std::string("cannot open ") + path + " for writing");
        const uint32_t version = dtype == 0 ? 1u : 2u;
        const uint64_t nn = (uint64_t)n, rr = (uint64_t)r;
        bool ok = std::fwrite("ROMB", 1, 4, out.f) == 4 && std::fwrite(&version, 4, 1, out.f) == 1 &&
                  std::fwrite(&nn, 8, 1, out.f) == 1 && std::fwrite(&rr, 8, 1, out.f) == 1;
        if (version == 2) {
            const uint8_t dt = (uint8_t)dtype;
            ok = ok && std::fwrite(&dt, 1, 1, out.f) == 1;
        }
        const size_t bytes = esize(dtype) * (size_t)n * (size_t)r;
        if (where == 1) {
            std::vector<char> h(std::min(bytes, kRombChunk));
            for (size_t o = 0; ok && o < bytes; o += kRombChunk) {
                const size_t b = std::min(kRombChunk, bytes - o);
                CK(cudaMemcpyAsync(h.data(), (const char*)V + o, b, cudaMemcpyDeviceToHost, ctx->c.s));
                ctx->c.sync();
                ok = std::fwrite(h.data(), 1, b, out.f) == b;
            }
        } else if (bytes) {
            ok = ok && std::fwrite(V, 1, bytes, out.f) == bytes;
        }
        if (r) ok = ok && std::fwrite(markers, 1, (size_t)r, out.f) == (size_t)r;
        if (!ok || std::fflush(out.f) != 0) throw rd::IoError(std::string("write failed: ") + path);
    });
}

int rd_romb_info(const char* path, int* dtype, long* n, long* r) {
    return guard([&] {
        File in(path, "rb");
        if (!in.f) throw rd::IoError(std::string("cannot open ") + path);
        const RombHeader h = romb_header(in.f, path);
        if (dtype) *dtype = h.dtype;
        if (n) *n = (long)h.n;
        if (r) *r = (long)h.r;
    });
}

int rd_romb_read(const char* path, int dtype, long n, long r, void* V, uint8_t* markers, int where, rd_ctx* ctx) {
    return guard([&] {
        if (where == 1 && !ctx) throw rd::ConfigError("romb: a context is needed for device data");
        File in(path, "rb");
        if (!in.f) throw rd::IoError(std::string("cannot open ") + path);
        const RombHeader h = romb_header(in.f, path);
        if (h.dtype != dtype || (long)h.n != n || (long)h.r != r)
            throw rd::ConfigError(std::string(path) + ": header does not match the requested dtype / shape");
        const size_t bytes = esize(dtype) * (size_t)n * (size_t)r;
        bool ok = true;
        if (where == 1) {
            std::vector<char> hb(std::min(bytes, kRombChunk));
            for (size_t o = 0; ok && o < bytes; o += kRombChunk) {
                const size_t b = std::min(kRombChunk, bytes - o);
                ok = std::fread(hb.data(), 1, b, in.f) == b;
                if (ok) {
                    CK(cudaMemcpyAsync((char*)V + o, hb.data(), b, cudaMemcpyHostToDevice, ctx->c.s));
                    ctx->c.sync();
                }
            }
        } else if (bytes) {
            ok = std::fread(V, 1, bytes, in.f) == bytes;
        }
        std::vector<uint8_t> mk((size_t)r);
        if (ok && r) ok = std::fread(mk.data(), 1, (size_t)r, in.f) == (size_t)r;
        if (!ok) throw rd::IoError(std::string(path) + ": truncated basis file");
        if (markers) std::memcpy(markers, mk.data(), (size_t)r);
    });
}

int rd_basis_save(rd_basis* b, const char* path) {
    return guard([&] {
        BASIS_DISPATCH(b, {
            const int rc = rd_romb_write(path, b->h.dtype, B.n, B.cols, B.Vp(), B.markers.data(), 1, b->ctx);
            if (rc == 4) throw rd::IoError(g_err);
            if (rc) throw std::runtime_error(g_err);
        });
    });
}

}  // extern "C"
