// TEST INFRASTRUCTURE ONLY.
//
// C entry points over the REFERENCE'S OWN functions (romdot:: in
// /root/reference/proj/src/*.cpp), so that tests
// can run the reference itself on the inputs the restatement
// (romdot_oracle.cpp) and the CUDA path get.  This file contains no
// algorithm: every ref_* function marshals plain arrays (column-major) into
// the reference's types and calls the reference function named in its
// comment.  Built by `make -C oracle _ref` into oracle/_ref/libromdot_ref.so
// together with the reference sources, which are compiled where they lie
// against oracle/eigen_shim (Eigen itself is absent from this image).
//
// Return codes follow the reference's taxonomy (tools/romdot.cpp:79-91):
// 0 ok, 2 ConfigError, 3 SolverError, 4 IoError, 1 anything else.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "romdot/basis.hpp"
#include "romdot/config.hpp"
#include "romdot/grid.hpp"
#include "romdot/harness.hpp"
#include "romdot/inversion.hpp"
#include "romdot/io.hpp"
#include "romdot/krylov.hpp"
#include "romdot/pals.hpp"
#include "romdot/rom.hpp"

using namespace romdot;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const SolverError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

Vec vec_in(const double* p, long n) {
    Vec v(n);
    std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(n));
    return v;
}
Mat mat_in(const double* p, long r, long c) {
    Mat m(r, c);
    if (r * c > 0) std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(r * c));
    return m;
}
void out(const Mat& m, double* p) {
    if (p && m.size() > 0) std::memcpy(p, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
}

struct RefGrid {
    Grid grid;
    BlockSystem blocks;
    SchurOperator op;
    SourceDetectorLayout layout;
    bool has_layout = false;
    explicit RefGrid(const GridConfig& cfg) : grid(cfg), blocks(assemble_blocks(grid)), op(grid, blocks) {}
};

struct RefBasis {
    InitBasisResult init;
};

struct RefRecycler {
    std::unique_ptr<BaselinePerRhsRecycler> r;
};

struct RefRom {
    std::unique_ptr<ReducedModel> rom;
};

PalsModel pals_in(int m_bumps, const double* prm) {
    PalsModel m;
    m.m_bumps = m_bumps;
    m.mu_in = prm[0];
    m.mu_out = prm[1];
    m.eps_heaviside = prm[2];
    m.eps_norm = prm[3];
    m.level = prm[4];
    return m;
}

// ExperimentConfig with the reference's defaults (config.hpp:33-63) and the
// fields acceptance.cpp / harness.cpp set: c = {nx, ny, n_src, n_det, m_bumps,
// seed, k_systems, k_eig, tol_basis}; a negative entry keeps the default.
ExperimentConfig exp_in(const double* c) {
    ExperimentConfig cfg;
    if (c[0] >= 0) cfg.grid.nx = static_cast<int>(c[0]);
    if (c[1] >= 0) cfg.grid.ny = static_cast<int>(c[1]);
    if (c[2] >= 0) cfg.n_src = static_cast<int>(c[2]);
    if (c[3] >= 0) cfg.n_det = static_cast<int>(c[3]);
    if (c[4] >= 0) cfg.pals.m_bumps = static_cast<int>(c[4]);
    if (c[5] >= 0) cfg.run.seed = static_cast<std::uint64_t>(c[5]);
    if (c[6] >= 0) cfg.run.k_systems = static_cast<int>(c[6]);
    if (c[7] >= 0) cfg.run.k_eig = static_cast<int>(c[7]);
    if (c[8] >= 0) cfg.run.tol_basis = c[8];
    return cfg;
}

struct RefHybrid {
    ExperimentConfig cfg;
    std::unique_ptr<Problem> prob;
    std::unique_ptr<HybridEvaluator> eval;
};

void log_out(const ProcessResult& res, double* X, double* log, long* its, long* appends) {
    out(res.X, X);
    for (std::size_t t = 0; t < res.log.size(); ++t) {
        const BuildLogRow& r = res.log[t];
        double* row = log + 5 * t;
        row[0] = r.system;
        row[1] = r.rhs;
        row[2] = r.init_relres;
        row[3] = r.iterations;
        row[4] = r.appended ? 1.0 : 0.0;
    }
    *its = res.inner_iterations;
    *appends = res.appends;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Grid + assemble_blocks + SchurOperator (grid.cpp:9-93)
void* ref_grid_create(int nx, int ny, double a1, double b1, double a3, double b3, double diffusion,
                      double boundary_constant) {
    RefGrid* g = nullptr;
    guard([&] {
        GridConfig cfg;
        cfg.nx = nx;
        cfg.ny = ny;
        cfg.a1 = a1;
        cfg.b1 = b1;
        cfg.a3 = a3;
        cfg.b3 = b3;
        cfg.diffusion = diffusion;
        cfg.boundary_constant = boundary_constant;
        g = new RefGrid(cfg);
    });
    return g;
}
void ref_grid_free(void* g) { delete static_cast<RefGrid*>(g); }
long ref_grid_dim(void* g) { return static_cast<RefGrid*>(g)->op.dim(); }
double ref_grid_h(void* g) { return static_cast<RefGrid*>(g)->grid.h(); }
// Grid::interior_nodes (grid.cpp:27-36), n x 2
int ref_grid_interior_nodes(void* g, double* nodes) {
    return guard([&] { out(static_cast<RefGrid*>(g)->grid.interior_nodes(), nodes); });
}
// SchurOperator::apply (grid.cpp:95-97)
int ref_apply(void* g, const double* mu, const double* x, double* y) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        const long n = G->op.dim();
        out(G->op.apply(vec_in(mu, n), vec_in(x, n)), y);
    });
}
// SchurOperator::with_absorption (grid.cpp:99-105), dense n x n
int ref_with_absorption_dense(void* g, const double* mu, double* A) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        out(Mat(G->op.with_absorption(vec_in(mu, G->op.dim()))), A);
    });
}
// full_block_matrix (grid.cpp:162-173), (nb+ni)^2
int ref_full_block_matrix(void* g, const double* mu, double* A) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        out(full_block_matrix(G->grid, G->blocks, vec_in(mu, G->op.dim())), A);
    });
}
// evenly_spaced_positions (grid.cpp:107-121)
int ref_evenly_spaced(int nx, int count, int* pos) {
    return guard([&] {
        const std::vector<int> p = evenly_spaced_positions(nx, count);
        std::memcpy(pos, p.data(), sizeof(int) * p.size());
    });
}
// effective_layout (grid.cpp:123-160); B_concat n x (ns+nd)
int ref_layout(void* g, int ns, const int* spos, int nd, const int* dpos, double* Bconcat) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        G->layout = effective_layout(G->grid, G->blocks, std::vector<int>(spos, spos + ns),
                                     std::vector<int>(dpos, dpos + nd));
        G->has_layout = true;
        out(G->layout.B_concat, Bconcat);
    });
}

// minres (krylov.cpp:100-104)
int ref_minres(void* g, const double* mu, const double* b, double tol, int maxit, double* x, int* its, int* conv,
               double* hist, long cap, long* hl) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        const long n = G->op.dim();
        const Vec m = vec_in(mu, n);
        const LinOp apply = [&](const Vec& v) { return G->op.apply(m, v); };
        auto [sol, rep] = minres(apply, vec_in(b, n), tol, maxit);
        out(sol, x);
        *its = rep.iterations;
        *conv = rep.converged ? 1 : 0;
        *hl = static_cast<long>(rep.rel_residual_history.size());
        for (long i = 0; i < std::min(cap, *hl); ++i) hist[i] = rep.rel_residual_history[static_cast<std::size_t>(i)];
    });
}
// minres on a dense symmetric matrix (test_krylov.cpp's indefinite cases)
int ref_minres_dense(long n, const double* A, const double* b, double tol, int maxit, double* x, int* its,
                     int* conv, double* hist, long cap, long* hl) {
    return guard([&] {
        const Mat M = mat_in(A, n, n);
        const LinOp apply = [&](const Vec& v) { return Vec(M * v); };
        auto [sol, rep] = minres(apply, vec_in(b, n), tol, maxit);
        out(sol, x);
        *its = rep.iterations;
        *conv = rep.converged ? 1 : 0;
        *hl = static_cast<long>(rep.rel_residual_history.size());
        for (long i = 0; i < std::min(cap, *hl); ++i) hist[i] = rep.rel_residual_history[static_cast<std::size_t>(i)];
    });
}
// RecycleSpace::from_raw (krylov.cpp:106-115)
int ref_from_raw(long n, long c, const double* W, const double* AW, double* U, double* K) {
    return guard([&] {
        const RecycleSpace rs = RecycleSpace::from_raw(mat_in(W, n, c), mat_in(AW, n, c));
        out(rs.U(), U);
        out(rs.K(), K);
    });
}
// from_raw + RecycleSpace::append (krylov.cpp:117-139); U, K hold c+1 columns
int ref_from_raw_append(long n, long c, const double* W, const double* AW, const double* u, const double* k,
                        double* U, double* K, int* appended) {
    return guard([&] {
        RecycleSpace rs = RecycleSpace::from_raw(mat_in(W, n, c), mat_in(AW, n, c));
        *appended = rs.append(vec_in(u, n), vec_in(k, n)) ? 1 : 0;
        out(rs.U(), U);
        out(rs.K(), K);
    });
}
// initial_guess (krylov.cpp:141-145)
int ref_initial_guess(long n, long c, const double* W, const double* AW, const double* b, double* z, double* r) {
    return guard([&] {
        const RecycleSpace rs = RecycleSpace::from_raw(mat_in(W, n, c), mat_in(AW, n, c));
        auto [zz, rr] = initial_guess(rs, vec_in(b, n));
        out(zz, z);
        out(rr, r);
    });
}
// recycled_minres (krylov.cpp:147-179)
int ref_recycled_minres(void* g, const double* mu, long c, const double* W, const double* AW, const double* rhs,
                        double tol, int maxit, double rhs_scale, double* corr, double* nd, double* image, int* its,
                        int* conv, double* corr_norm, double* hist, long cap, long* hl) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        const long n = G->op.dim();
        const Vec m = vec_in(mu, n);
        const LinOp apply = [&](const Vec& v) { return G->op.apply(m, v); };
        const RecycleSpace rs = RecycleSpace::from_raw(mat_in(W, n, c), mat_in(AW, n, c));
        const RecycledResult res = recycled_minres(apply, rs, vec_in(rhs, n), tol, maxit, rhs_scale);
        out(res.correction, corr);
        out(res.new_direction, nd);
        out(res.image, image);
        *its = res.report.iterations;
        *conv = res.report.converged ? 1 : 0;
        *corr_norm = res.report.correction_norm;
        *hl = static_cast<long>(res.report.rel_residual_history.size());
        for (long i = 0; i < std::min(cap, *hl); ++i)
            hist[i] = res.report.rel_residual_history[static_cast<std::size_t>(i)];
    });
}
// smallest_eigenpairs (krylov.cpp:181-280) on with_absorption(mu)
int ref_smallest_eigenpairs(void* g, const double* mu, int k, double tol, double* lam, double* U) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        auto [l, u] = smallest_eigenpairs(G->op.with_absorption(vec_in(mu, G->op.dim())), k, tol);
        out(l, lam);
        out(u, U);
    });
}

// init_basis (basis.cpp:136-155)
void* ref_init_basis(void* g, const double* mu0, const double* B, long nrhs, int k_eig, double tol) {
    RefBasis* b = nullptr;
    guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        const long n = G->op.dim();
        auto nb = std::make_unique<RefBasis>();
        nb->init = init_basis(G->op, vec_in(mu0, n), mat_in(B, n, nrhs), k_eig, tol);
        b = nb.release();
    });
    return b;
}
// init_basis_from (basis.cpp:114-134)
void* ref_init_basis_from(void* g, const double* U0, long ku, const double* X0, long nrhs) {
    RefBasis* b = nullptr;
    guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        const long n = G->op.dim();
        auto nb = std::make_unique<RefBasis>();
        nb->init = init_basis_from(G->op, mat_in(U0, n, ku), mat_in(X0, n, nrhs));
        b = nb.release();
    });
    return b;
}
void ref_basis_free(void* b) { delete static_cast<RefBasis*>(b); }
long ref_basis_cols(void* b) { return static_cast<RefBasis*>(b)->init.basis.cols(); }
long ref_basis_ku(void* b) { return static_cast<RefBasis*>(b)->init.basis.eig_block(); }
long ref_basis_full_solves(void* b) { return static_cast<RefBasis*>(b)->init.full_solves; }
// which: 0 V, 1 K_img, 2 R, 3 K_raw, 4 Astar_V, 5 X0, 6 eigenvalues
int ref_basis_get(void* b, int which, double* p) {
    return guard([&] {
        const InitBasisResult& I = static_cast<RefBasis*>(b)->init;
        switch (which) {
            case 0: out(I.basis.V(), p); break;
            case 1: out(I.basis.K_img(), p); break;
            case 2: out(I.basis.R(), p); break;
            case 3: out(I.basis.K_raw(), p); break;
            case 4: out(I.basis.Astar_V(), p); break;
            case 5: out(I.X0, p); break;
            case 6: out(I.eigenvalues, p); break;
            default: throw ConfigError("ref_basis_get: bad selector");
        }
    });
}
void ref_basis_markers(void* b, std::uint8_t* m) {
    const auto& mk = static_cast<RefBasis*>(b)->init.basis.markers();
    std::memcpy(m, mk.data(), mk.size());
}
long ref_basis_space(void* b, long j, int* idx) {
    const auto& c = static_cast<RefBasis*>(b)->init.spaces.cols[static_cast<std::size_t>(j)];
    if (idx) std::memcpy(idx, c.data(), sizeof(int) * c.size());
    return static_cast<long>(c.size());
}
// GlobalBasis::refresh (basis.cpp:37-76)
int ref_basis_refresh(void* b, const double* mu) {
    return guard([&] {
        GlobalBasis& gb = static_cast<RefBasis*>(b)->init.basis;
        gb.refresh(vec_in(mu, gb.dim()));
    });
}
// GlobalBasis::append (basis.cpp:78-103)
int ref_basis_append(void* b, const double* y, const double* Astar_y, const double* mu, int marker, int* appended) {
    return guard([&] {
        GlobalBasis& gb = static_cast<RefBasis*>(b)->init.basis;
        const long n = gb.dim();
        *appended = gb.append(vec_in(y, n), vec_in(Astar_y, n), vec_in(mu, n), static_cast<std::uint8_t>(marker)) ? 1 : 0;
    });
}
// GlobalBasis::solve_projected / projected_coordinates (basis.cpp:105-112)
int ref_basis_solve_projected(void* b, const double* rhs, double* x, double* coords) {
    return guard([&] {
        const GlobalBasis& gb = static_cast<RefBasis*>(b)->init.basis;
        const Vec r = vec_in(rhs, gb.dim());
        out(gb.solve_projected(r), x);
        out(gb.projected_coordinates(r), coords);
    });
}
// process_system (basis.cpp:157-207); log rows: system, rhs, init_relres, iterations, appended
int ref_process_system(void* b, void* g, const double* mu, const double* B, long nrhs, double tol, int system_index,
                       int maxit, double* X, double* log, long* its, long* appends) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        auto* P = static_cast<RefBasis*>(b);
        const long n = G->op.dim();
        const ProcessResult res = process_system(P->init.basis, P->init.spaces, G->op, vec_in(mu, n),
                                                 mat_in(B, n, nrhs), tol, system_index, maxit);
        log_out(res, X, log, its, appends);
    });
}
// BaselinePerRhsRecycler (basis.cpp:209-266)
void* ref_recycler_create(void* g, const double* U0, long ku, const double* X0, long nrhs) {
    RefRecycler* r = nullptr;
    guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        const long n = G->op.dim();
        auto nr = std::make_unique<RefRecycler>();
        nr->r = std::make_unique<BaselinePerRhsRecycler>(G->op, mat_in(U0, n, ku), mat_in(X0, n, nrhs));
        r = nr.release();
    });
    return r;
}
void ref_recycler_free(void* r) { delete static_cast<RefRecycler*>(r); }
int ref_recycler_solve_system(void* r, long n, const double* mu, const double* B, long nrhs, double tol,
                              int system_index, int maxit, double* X, double* log, long* its, long* appends) {
    return guard([&] {
        const ProcessResult res = static_cast<RefRecycler*>(r)->r->solve_system(vec_in(mu, n), mat_in(B, n, nrhs), tol,
                                                                              system_index, maxit);
        log_out(res, X, log, its, appends);
    });
}
// basis_coefficients (basis.cpp:268-275)
int ref_basis_coefficients(long n, long r, const double* V, long m, const double* X, double* Cout) {
    return guard([&] { out(basis_coefficients(mat_in(V, n, r), mat_in(X, n, m)), Cout); });
}

// ReducedModel (rom.cpp:9-34); needs ref_layout first
void* ref_rom_create(void* g, const double* V, long r) {
    RefRom* m = nullptr;
    guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        if (!G->has_layout) throw ConfigError("ref_rom_create: call ref_layout first");
        auto nm = std::make_unique<RefRom>();
        nm->rom = std::make_unique<ReducedModel>(mat_in(V, G->op.dim(), r), G->op.matrix(), G->layout.B_tilde,
                                                 G->layout.C_tilde);
        m = nm.release();
    });
    return m;
}
void ref_rom_free(void* m) { delete static_cast<RefRom*>(m); }
// ReducedModel::reduced_system (rom.cpp:22-27), r x r
int ref_rom_reduced_system(void* m, long n, const double* mu, double* Ar) {
    return guard([&] { out(static_cast<RefRom*>(m)->rom->reduced_system(vec_in(mu, n)), Ar); });
}
// ReducedModel::transfer (rom.cpp:29-35), n_det x n_src
int ref_rom_transfer(void* m, long n, const double* mu, double* T) {
    return guard([&] { out(static_cast<RefRom*>(m)->rom->transfer(vec_in(mu, n)), T); });
}
// ReducedModel::jacobian (rom.cpp:37-67), (n_src n_det) x n_params
int ref_rom_jacobian(void* m, int m_bumps, const double* prm, const double* p, long n, const double* nodes, double h2,
                     double* J) {
    return guard([&] {
        const PalsModel pm = pals_in(m_bumps, prm);
        out(static_cast<RefRom*>(m)->rom->jacobian(pm, vec_in(p, pm.n_params()), mat_in(nodes, n, 2), h2), J);
    });
}
// fom_transfer (rom.cpp:94-98); mode 0 Direct, 1 Minres
int ref_fom_transfer(void* g, const double* mu, int mode, double tol, double* T) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        if (!G->has_layout) throw ConfigError("ref_fom_transfer: call ref_layout first");
        out(fom_transfer(G->op, G->layout, vec_in(mu, G->op.dim()), mode ? FomSolve::Minres : FomSolve::Direct, tol), T);
    });
}
// fom_jacobian (rom.cpp:122-129)
int ref_fom_jacobian(void* g, int m_bumps, const double* prm, const double* p, const double* nodes, double h2,
                     int mode, double tol, double* J) {
    return guard([&] {
        auto* G = static_cast<RefGrid*>(g);
        if (!G->has_layout) throw ConfigError("ref_fom_jacobian: call ref_layout first");
        const PalsModel pm = pals_in(m_bumps, prm);
        out(fom_jacobian(G->op, G->layout, pm, vec_in(p, pm.n_params()), mat_in(nodes, G->op.dim(), 2), h2,
                         mode ? FomSolve::Minres : FomSolve::Direct, tol),
            J);
    });
}

// eval_absorption (pals.cpp:66-75); prm = {mu_in, mu_out, eps_heaviside, eps_norm, level}
int ref_pals_absorption(int m_bumps, const double* prm, const double* p, long n, const double* nodes, double* mu) {
    return guard([&] {
        const PalsModel pm = pals_in(m_bumps, prm);
        out(eval_absorption(pm, vec_in(p, pm.n_params()), mat_in(nodes, n, 2)), mu);
    });
}
// absorption_jacobian (pals.cpp:77-129) as a dense column
int ref_pals_jacobian_column(int m_bumps, const double* prm, const double* p, int k, long n, const double* nodes,
                             double* col) {
    return guard([&] {
        const PalsModel pm = pals_in(m_bumps, prm);
        out(absorption_jacobian(pm, vec_in(p, pm.n_params()), k, mat_in(nodes, n, 2)).dense(static_cast<int>(n)), col);
    });
}

// ---- experiment layer (config.cpp, harness.cpp, io.cpp, inversion.cpp) ----

// sizes of the experiment's problem: {n, n_rhs, n_params}
int ref_exp_dims(const double* c, long* dims) {
    return guard([&] {
        const ExperimentConfig cfg = exp_in(c);
        Problem prob(cfg);
        dims[0] = prob.op.dim();
        dims[1] = prob.layout.n_src + prob.layout.n_det;
        dims[2] = cfg.pals.n_params();
    });
}
// parameter_in_sequence (harness.cpp:62-75) over ExperimentConfig::initial_parameters (config.cpp:163-184)
int ref_exp_parameters(const double* c, int index, double* p) {
    return guard([&] { out(parameter_in_sequence(exp_in(c), index), p); });
}
// mu = h2 * eval_absorption(pals, p_index, nodes) exactly as cmd_compare_recycling forms it (harness.cpp:213,226),
// and B_concat of the experiment's layout
int ref_exp_mu(const double* c, int index, double* mu, double* Bconcat) {
    return guard([&] {
        const ExperimentConfig cfg = exp_in(c);
        Problem prob(cfg);
        const Vec p = parameter_in_sequence(cfg, index);
        out(Vec(prob.h2 * eval_absorption(cfg.pals, p, prob.nodes)), mu);
        out(prob.layout.B_concat, Bconcat);
    });
}
// cmd_compare_recycling (harness.cpp:208-251): the body of acceptance criterion 5 (acceptance.cpp:314-334)
int ref_compare_recycling(const double* c, const char* out_dir, long* ours, long* baseline) {
    return guard([&] {
        const CompareTotals t = cmd_compare_recycling(exp_in(c), out_dir);
        *ours = t.ours;
        *baseline = t.baseline;
    });
}
// NormalStream (config.cpp:249-271)
int ref_normal_stream(std::uint64_t seed, long count, double* outv) {
    return guard([&] {
        NormalStream s(seed);
        for (long i = 0; i < count; ++i) outv[i] = s.next();
    });
}
// ExperimentConfig::offline_hash (config.cpp)
int ref_offline_hash(const double* c, char* buf, long cap) {
    return guard([&] {
        const std::string h = exp_in(c).offline_hash();
        std::strncpy(buf, h.c_str(), static_cast<std::size_t>(cap - 1));
        buf[cap - 1] = 0;
    });
}
// format_sci (io.cpp)
int ref_format_sci(double v, char* buf, long cap) {
    return guard([&] {
        const std::string h = format_sci(v);
        std::strncpy(buf, h.c_str(), static_cast<std::size_t>(cap - 1));
        buf[cap - 1] = 0;
    });
}
// write_basis / read_basis (io.cpp:77-131): the ROMB v1 file
int ref_write_basis(const char* path, long n, long r, const double* V, const std::uint8_t* markers) {
    return guard([&] { write_basis(path, mat_in(V, n, r), std::vector<std::uint8_t>(markers, markers + r)); });
}
int ref_read_basis(const char* path, long* n, long* r, double* V, std::uint8_t* markers) {
    return guard([&] {
        auto [M, mk] = read_basis(path);
        *n = M.rows();
        *r = M.cols();
        if (V) out(M, V);
        if (markers) std::memcpy(markers, mk.data(), mk.size());
    });
}

// HybridEvaluator (inversion.cpp:53-106) over init_basis at p0 = parameter_in_sequence(cfg, 0)
void* ref_hybrid_create(const double* c) {
    RefHybrid* h = nullptr;
    guard([&] {
        auto nh = std::make_unique<RefHybrid>();
        nh->cfg = exp_in(c);
        nh->prob = std::make_unique<Problem>(nh->cfg);
        const Problem& prob = *nh->prob;
        const Vec p0 = parameter_in_sequence(nh->cfg, 0);
        const Vec mu0 = prob.h2 * eval_absorption(nh->cfg.pals, p0, prob.nodes);
        auto init = init_basis(prob.op, mu0, prob.layout.B_concat, nh->cfg.run.k_eig, nh->cfg.run.tol_basis);
        ForwardSetup fs;
        fs.op = &prob.op;
        fs.layout = &prob.layout;
        fs.pals = &nh->cfg.pals;
        fs.nodes = prob.nodes;
        fs.h2 = prob.h2;
        nh->eval = std::make_unique<HybridEvaluator>(fs, std::move(init), p0, nh->cfg.run.k_systems,
                                                     nh->cfg.run.tol_basis);
        h = nh.release();
    });
    return h;
}
void ref_hybrid_free(void* h) { delete static_cast<RefHybrid*>(h); }
// HybridEvaluator::transfer (inversion.cpp:82-95), n_det x n_src
int ref_hybrid_transfer(void* h, const double* p, double* T) {
    return guard([&] {
        auto* H = static_cast<RefHybrid*>(h);
        out(H->eval->transfer(vec_in(p, H->cfg.pals.n_params())), T);
    });
}
// HybridEvaluator::jacobian (inversion.cpp:97-105)
int ref_hybrid_jacobian(void* h, const double* p, double* J) {
    return guard([&] {
        auto* H = static_cast<RefHybrid*>(h);
        out(H->eval->jacobian(vec_in(p, H->cfg.pals.n_params())), J);
    });
}
// state: {basis cols, systems_used, appends, in_rom_mode, full_order_solves, log rows}
int ref_hybrid_state(void* h, long* st) {
    return guard([&] {
        auto* H = static_cast<RefHybrid*>(h);
        st[0] = H->eval->basis().cols();
        st[1] = H->eval->systems_used();
        st[2] = H->eval->appends();
        st[3] = H->eval->in_rom_mode() ? 1 : 0;
        st[4] = H->eval->full_order_solves;
        st[5] = static_cast<long>(H->eval->build_log().size());
    });
}
int ref_hybrid_log(void* h, double* log) {
    return guard([&] {
        auto* H = static_cast<RefHybrid*>(h);
        const auto& L = H->eval->build_log();
        for (std::size_t t = 0; t < L.size(); ++t) {
            double* row = log + 5 * t;
            row[0] = L[t].system;
            row[1] = L[t].rhs;
            row[2] = L[t].init_relres;
            row[3] = L[t].iterations;
            row[4] = L[t].appended ? 1.0 : 0.0;
        }
    });
}
int ref_hybrid_basis_V(void* h, double* V) {
    return guard([&] { out(static_cast<RefHybrid*>(h)->eval->basis().V(), V); });
}

}  // extern "C"
