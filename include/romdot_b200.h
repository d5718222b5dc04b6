/*
 * romdot_b200 -- C ABI of the B200-native recycled-Krylov global-basis builder.
 *
 * Plain pointers and sizes only; no torch, Eigen or CUDA types cross this
 * boundary. Every entry point returns an int status:
 *   0 OK, 2 config error (reference ConfigError), 3 solver error (reference
 *   SolverError: non-convergence, breakdown), 4 IO error, 5 CUDA error,
 *   1 other. rd_last_error() returns the message of the last failure on the
 *   calling thread. No C++ exception crosses this boundary.
 *
 * dtype: 0 = float64 (SPD systems, omega = 0), 1 = complex128 (interleaved
 * re/im; complex-symmetric systems, omega != 0).
 * where: 0 = host pointers (copied in / out inside the call),
 *        1 = device pointers (borrowed, never freed; stream-ordered).
 * Matrices are column-major with leading dimension n (the node count).
 *
 * The reference interface each entry point replaces is cited per function
 * (paths relative to the reference repository's proj/ directory).
 */
#ifndef ROMDOT_B200_H
#define ROMDOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rd_ctx rd_ctx;     /* device, stream, reduction workspace */
typedef struct rd_op rd_op;       /* Schur operator A~(p) on the device */
typedef struct rd_basis rd_basis; /* GlobalBasis + PerRhsSpaces on the device */
typedef struct rd_rom rd_rom;     /* ReducedModel: V and the reduced-system workspace */

typedef struct rd_report {
    int iterations;      /* SolveReport::iterations   (include/romdot/krylov.hpp:10-15) */
    int converged;       /* SolveReport::converged */
    double correction_norm;
    double final_relres;
} rd_report;

/* ------------------------------------------------------------ context --- */
int rd_ctx_create(int device, rd_ctx** out);
void rd_ctx_destroy(rd_ctx* ctx);
const char* rd_last_error(void);
int rd_ctx_sync(rd_ctx* ctx);
/* Device time (ms) between the last two rd_ctx_mark() calls (CUDA events on the ctx stream). */
int rd_ctx_mark(rd_ctx* ctx);
double rd_ctx_elapsed_ms(rd_ctx* ctx);
/* Number of this library's kernel launches issued on the context so far. */
long rd_ctx_launches(rd_ctx* ctx);
/* Inner solver of every entry point below that solves (rd_recycled_solve,
 * rd_initial_solutions, rd_process_system, rd_per_rhs_solve_system):
 *   0  recycled CG / COCG, device-resident recurrence (default; the hot path);
 *   1  the reference's recycled MINRES (src/krylov.cpp:17-98 minres_core,
 *      :147-179 recycled_minres) with its stopping rules -- real operators only
 *      (ConfigError, status 2, for complex data). Parity path: reproduces the
 *      reference's BuildLog iteration counts; scalar recurrence on the host.   */
int rd_ctx_set_solver(rd_ctx* ctx, int solver);
int rd_ctx_get_solver(rd_ctx* ctx);
/* Sampled per-kernel-class device timing of the inner iteration (CUDA events on
 * the ctx stream, first iteration of each launch batch). enable resets the counters.
 * cls: 0 cg_stencil_dots, 1 ts_T, 2 ts_NT, 3 cg_update, 4 cg_fused (one event
 * pair around a batch of back-to-back launches), 5 one step of the batched
 * iteration (seven launches; samples = steps), 6 the same time with samples =
 * slot-steps (inner iterations done by the batched path). bytes = algorithmic. */
void rd_ctx_profile(rd_ctx* ctx, int enable);
int rd_ctx_prof_get(rd_ctx* ctx, int cls, double* ms, double* bytes, long* samples);
/* ROMDOT_FUSED_CHECK=1 (debug): cg_fused stamps each row tile with the launch's
 * epoch when its r' rows are published, and every stencil halo read checks the
 * stamps of the tiles it reads after acquiring the step counters -- a race
 * detector for the cross-CTA protocol (a violation fails the solve, status 3).
 * Totals over the context: fused launches checked and stale reads seen.     */
void rd_ctx_fused_check(rd_ctx* ctx, long* launches_checked, long* violations);
/* Raw stream handle (cudaStream_t) for interop. */
void* rd_ctx_stream(rd_ctx* ctx);

/* ----------------------------------------------------------- operator --- */
/* Replaces SchurOperator (include/romdot/grid.hpp:100-114, src/grid.cpp:86-105)
 * and the LinOp plug-in (include/romdot/types.hpp:18). d = 2 or 3; N[d-1] is
 * the Robin axis. robin_face = Dbg/(1+rho), rho = 2*A*Dbg/h.                 */
int rd_op_create(rd_ctx* ctx, int d, const long* N, double robin_face, rd_op** out);
void rd_op_destroy(rd_op* op);
/* Per-system coefficient fields: node D, h^2 mu_a, shift = h^2 omega/nu.
 * Replaces the mu_scaled argument of SchurOperator::apply (src/grid.cpp:95). */
int rd_op_set_fields(rd_op* op, const double* D, const double* mu, double shift, int where);
/* y[:, j] = A x[:, j], j < ncols (SchurOperator::apply, src/grid.cpp:95-97). */
int rd_op_apply(rd_op* op, int dtype, const void* x, void* y, long ncols, int where);
double rd_op_lam_max(rd_op* op); /* Gershgorin bound (src/krylov.cpp:190-195) */

/* ------------------------------------------------------------ solvers --- */
/* Recycled CG / COCG on the correction equation with recycle space (U, K),
 * A U = K, K^T K = I (bilinear for complex). c = 0: plain CG / COCG.
 * Replaces recycled_minres (include/romdot/krylov.hpp:57-58, src/krylov.cpp:147-179)
 * and minres (krylov.hpp:44): convergence ||rhs - A g|| / rhs_scale <= tol.
 * Outputs: g (correction), y (new direction y_m), image (A y_m).
 * hist (optional, hist_cap entries) receives the relative residual history.  */
int rd_recycled_solve(rd_op* op, int dtype, const void* U, const void* K, long c, const void* rhs, double tol,
                      long maxit, double rhs_scale, void* g, void* y, void* image, rd_report* rep, double* hist,
                      long hist_cap, int where);
/* RecycleSpace::from_raw (src/krylov.cpp:106-115): K = orth(AW) (bilinear for
 * complex), U = W R^-1. Writes U, K (n x c). */
int rd_recycle_space_from_raw(rd_ctx* ctx, int dtype, long n, long c, const void* W, const void* AW, void* U,
                              void* K, int where);

/* X0 of init_basis (src/basis.cpp:141-149): one CG/COCG solve per column of
 * B_concat (one nonzero per column: bidx, bval) at 0.25 * tol, maxit = 2n.   */
int rd_initial_solutions(rd_op* op, int dtype, long nrhs, const long* bidx, const double* bval, double tol,
                         void* X0, int where, long* total_iterations);

/* smallest_eigenpairs (src/krylov.cpp:181-280): k smallest eigenpairs of the
 * real SPD operator (fields at omega = 0), shift-invert Lanczos with inner CG. */
int rd_smallest_eigenpairs(rd_op* op, long k, double tol, double* lambda, void* U, int where);

/* -------------------------------------------------------- global basis --- */
/* init_basis_from (src/basis.cpp:114-134): V = [U0, X0], markers, per-RHS
 * spaces. cap = candidate-column cap (0 = unbounded).                       */
int rd_basis_create(rd_ctx* ctx, int dtype, long n, long ku, long nrhs, const void* U0, const void* X0, long cap,
                    int where, rd_basis** out);
void rd_basis_destroy(rd_basis* b);
long rd_basis_cols(rd_basis* b);
long rd_basis_eig_block(rd_basis* b);
/* Correction solves of rd_process_system / rd_per_rhs_solve_system that ran in the
 * batched iteration so far (8 independent right-hand sides of a system in flight,
 * the system's eigen block streamed once for all of them): the right-hand sides
 * after the candidate cap stopped the appends, where the reference's loop
 * (src/basis.cpp:168-205) leaves them independent. ROMDOT_BATCH=0 disables it. */
long rd_basis_batched_solves(rd_basis* b);
/* 1 once the image factor (K_img, R, W) exists, i.e. after the first refresh;
 * before it the reference's Kimg_/R_ are empty (include/romdot/basis.hpp:63). */
int rd_basis_factored(rd_basis* b);
/* which: 0 V, 1 K_img, 2 R (cols x cols), 3 W = V R^-1. Host output.
 * which != 0 before the first refresh: status 2 (no image factor yet). */
int rd_basis_get(rd_basis* b, int which, void* out);
/* Device pointer of V / K_img / W (valid until the next call that grows the basis).
 * W = V R^-1 is formed lazily: the columns appended since the last refresh / X
 * assembly are formed by this call (which >= 2) and by rd_basis_get(which = 3);
 * a W pointer taken before later appends does not see their columns formed.
 * Returns NULL (rd_last_error set) for W before the first refresh or after
 * rd_basis_compress, and on any CUDA failure while forming W.               */
void* rd_basis_device_ptr(rd_basis* b, int which);
/* Checkpoint hook (test / baseline instrumentation; no reference counterpart):
 * rd_process_system calls fn(user, system_index, j) before RHS j, with the
 * stream idle, so fn may read the state the reference's loop body
 * (src/basis.cpp:168-205) starts RHS j from -- V, K_img, R (rd_basis_get) and
 * U_j (rd_basis_space). A nonzero return aborts the system with status 3.
 * fn = NULL removes the hook.                                                */
int rd_basis_set_rhs_hook(rd_basis* b, int (*fn)(void* user, int system_index, long rhs), void* user);
int rd_basis_markers(rd_basis* b, uint8_t* out);
long rd_basis_space(rd_basis* b, long j, int* out);
/* GlobalBasis::refresh (src/basis.cpp:37-76) for the operator's current fields. */
int rd_basis_refresh(rd_basis* b, rd_op* op);
/* GlobalBasis::append (src/basis.cpp:78-103); z = A_i y. *appended = 0|1.   */
int rd_basis_append(rd_basis* b, const void* y, const void* z, int marker, int where, int* appended);
/* solve_projected / projected_coordinates (src/basis.cpp:105-112).          */
int rd_basis_solve_projected(rd_basis* b, const void* rhs, void* x, void* coords, int where);
/* process_system (src/basis.cpp:157-207). log: nrhs rows x 5 doubles
 * {system, rhs, init_relres, iterations, appended} (BuildLogRow, basis.hpp:17-23).
 * X (n x nrhs) may be NULL.                                                  */
int rd_process_system(rd_basis* b, rd_op* op, long nrhs, const long* bidx, const double* bval, double tol,
                      int system_index, long maxit, void* X, int where, double* log, long* inner_iterations,
                      long* appends);

/* Explicit residuals ||b_j - A x_j|| / ||b_j|| of a solution block (the
 * test_basis.cpp:180-193 check, at any size). X is n x nrhs.               */
int rd_residual_norms(rd_op* op, int dtype, long nrhs, const long* bidx, const double* bval, const void* X, int where,
                      double* out);

/* ---------------------------------------------------------- compression --- */
/* Rank-revealing compression of the n x m candidate basis (acceptance.cpp:368-383
 * truncation rule, BASELINE RRQR): column-normalised (if normalize) pivoted QR
 * at relative tolerance tol. Outputs rank, perm (m), rdiag (m), Q (n x rank). */
int rd_rrqr(rd_ctx* ctx, int dtype, long n, long m, const void* A, double tol, int normalize, long* rank,
            long* perm, double* rdiag, void* Q, int where);
/* In-place Algorithm-1 compression of a finished build: frees the
 * factorisation workspace, RRQR on V's own buffer, V <- orthonormal Q
 * (n x rank). perm / rdiag have basis-cols entries. The basis is final.   */
int rd_basis_compress(rd_basis* b, double tol, int normalize, long* rank, long* perm, double* rdiag);

/* ------------------------------------------- per-RHS-only comparator --- */
/* BaselinePerRhsRecycler (include/romdot/basis.hpp:102-119, src/basis.cpp:
 * 209-266): each RHS recycles only its own space U_j = [U0, X0_j, own new
 * directions]; no global check, no cross-RHS sharing, inner solves at tol.
 * The handle is an rd_basis holding V and the per-RHS index lists only
 * (rd_basis_cols/get(0)/space work; refresh/append/process_system refuse it);
 * free it with rd_basis_destroy.                                            */
int rd_per_rhs_create(rd_ctx* ctx, int dtype, long n, long ku, long nrhs, const void* U0, const void* X0, int where,
                      rd_basis** out);
/* BaselinePerRhsRecycler::solve_system (basis.cpp:221-264): X (n x nrhs) and
 * the same 5-column log as rd_process_system.                              */
int rd_per_rhs_solve_system(rd_basis* b, rd_op* op, long nrhs, const long* bidx, const double* bval, double tol,
                            int system_index, long maxit, void* X, int where, double* log, long* inner_iterations,
                            long* appends);

/* -------------------------------------------------------- reduced model --- */
/* ReducedModel (include/romdot/rom.hpp:12-41, src/rom.cpp:9-67) on the device.
 * V (n x r, column-major) is copied for where = 0 and BORROWED for where = 1
 * (e.g. rd_basis_device_ptr of a compressed basis; it must outlive the rom).
 * The constructor's E_r = V^T V SPD check (rom.cpp:12-14) is the Cholesky of
 * V^H V: status 3 "basis is numerically rank deficient" when it fails.
 * Projections are bilinear (V^T A V, V^T B, V^T C) for complex bases, which
 * keeps the reduced system complex symmetric (SURVEY §8 hard parts).      */
int rd_rom_create(rd_ctx* ctx, int dtype, long n, long r, const void* V, int where, rd_rom** out);
void rd_rom_destroy(rd_rom* rom);
long rd_rom_order(rd_rom* rom);
/* E_r = V^T V (ReducedModel::E_r, rom.hpp:24), r x r.                     */
int rd_rom_E(rd_rom* rom, void* E, int where);
/* A_r(p) = sym(V^T A(p) V) for the operator's current fields
 * (ReducedModel::reduced_system, rom.cpp:21-27), r x r.                    */
int rd_rom_reduced_system(rd_rom* rom, rd_op* op, void* Ar, int where);
/* Psi_r = C_r^T A_r^-1 B_r, n_det x n_src (ReducedModel::transfer,
 * rom.cpp:29-35). B~ / C~ columns have one nonzero each (grid.cpp:146-158),
 * passed as host (index, value) pairs; LU with partial pivoting replaces the
 * LDLT (status 3 on a singular reduced system, like rom.cpp:32-33).        */
int rd_rom_transfer(rd_rom* rom, rd_op* op, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, void* Psi, int where);
/* Reduced Jacobian (ReducedModel::jacobian, rom.cpp:37-67): column k =
 * scale * vec(sum_t w_t (V Z)[i_t,:]^T (V Y)[i_t,:]) with Y = A_r^-1 B_r,
 * Z = A_r^-1 C_r and the k-th parameter's compact support (i_t, w_t) in CSR
 * form (sup_ptr[n_par+1], sup_idx, sup_val: absorption_jacobian's SparseDiag
 * lists). The reference's scale is -h^2. J is (n_det*n_src) x n_par.      */
int rd_rom_jacobian(rd_rom* rom, rd_op* op, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, long n_par, const long* sup_ptr, const long* sup_idx,
                    const double* sup_val, double scale, void* J, int where);

/* ----------------------------------------------------- full-order model --- */
/* fom_transfer (src/rom.cpp:86-91, FomSolve::Minres): Psi = C~^T A^-1 B~,
 * n_det x n_src, by batched independent CG (omega = 0) / COCG solves at
 * relative tolerance tol (the reference's default is 1e-10).               */
int rd_fom_transfer(rd_op* op, int dtype, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, double tol, void* Psi, int where,
                    long* total_iterations);
/* fom_jacobian / jacobian_from_solutions (src/rom.cpp:101-129): X = A^-1 B~,
 * Z = A^-1 C~ (one batched solve), column k = scale * vec(sum_t w_t
 * Z[i_t,:]^T X[i_t,:]) over the k-th CSR support; the reference's scale is
 * -h^2. J is (n_det*n_src) x n_par.                                        */
int rd_fom_jacobian(rd_op* op, int dtype, long n_src, const long* src_idx, const double* src_val, long n_det,
                    const long* det_idx, const double* det_val, long n_par, const long* sup_ptr, const long* sup_idx,
                    const double* sup_val, double scale, double tol, void* J, int where);

/* ------------------------------------------------------------- ROMB I/O --- */
/* Basis file (src/io.cpp:77-110, README.md:96-99): "ROMB", u32 version,
 * u64 n, u64 r, column-major data, r marker bytes (little-endian). dtype 0
 * writes the reference's version 1 bit-exactly; dtype 1 (complex128) writes
 * version 2, which adds one dtype byte after r. Errors are IoError (status 4):
 * cannot open, not a basis file, unsupported version, truncated, marker count
 * != column count (io.cpp:80-81). where = 1: V is device memory (ctx needed). */
int rd_romb_write(const char* path, int dtype, long n, long r, const void* V, const uint8_t* markers, int where,
                  rd_ctx* ctx);
/* Header only: dtype, n, r of a version 1 or 2 file.                       */
int rd_romb_info(const char* path, int* dtype, long* n, long* r);
/* read_basis (io.cpp:93-110) into V (n x r, host or device) and markers (r).
 * The dtype / shape must match the header (rd_romb_info).                  */
int rd_romb_read(const char* path, int dtype, long n, long r, void* V, uint8_t* markers, int where, rd_ctx* ctx);
/* write_basis of a device basis: V and its markers (harness.cpp:194).      */
int rd_basis_save(rd_basis* b, const char* path);

/* ------------------------------------------------------- bench hooks --- */
/* Mean device ms per launch of the three inner-iteration projection kernels
 * (ms_out[0] c = K^T x, [1] fused x' = x - K c1 ; c2 = K^T x', [2] update)
 * on a seeded random n x c basis, and of the multi-column stencil apply.    */
int rd_bench_projection(rd_ctx* ctx, int dtype, long n, long c, int iters, double* ms_out);
int rd_bench_stencil(rd_op* op, int dtype, long ncols, int iters, double* ms_out);
/* Mean device ms of the tall Gram X^T X (sym) or X^T Y on seeded n x a / n x b data. */
int rd_bench_gram(rd_ctx* ctx, int dtype, long n, long a, long b, int sym, int iters, double* ms_out);
/* Mean device ms of the tall GEMM Z = X M (n x a by a x b; upper: M upper
 * triangular, the refresh's S^-1 products) on seeded data.                 */
int rd_bench_gemm(rd_ctx* ctx, int dtype, long n, long a, long b, int upper, int iters, double* ms_out);

#ifdef __cplusplus
}
#endif

#endif /* ROMDOT_B200_H */
