"""Generate tests/golden/ref_*.npz by running THE REFERENCE ITSELF
(oracle/_ref/libromdot_ref.so = /root/reference/proj/src/*.cpp compiled
unmodified against oracle/eigen_shim, see oracle/ref.py) on the reference's
own problems.  Needs /root/reference (this container); the fixtures travel.

    python scripts/make_ref_golden.py            # all fixtures

Fixtures (inputs + the reference's outputs; nothing here is computed by the
restatement or the CUDA path):
  ref_desk.npz        test_basis.cpp's Desk(21, 4, 4) with its PaLS params(offset): operator
                      apply, MINRES history, eigenpairs, init_basis, 4 x process_system
                      BuildLog + transfer functions, per-RHS-only recycler, ROM.
  ref_criterion5.npz  acceptance.cpp criterion 5 (121^2, 32 + 32, 9 bumps, seed 1234):
                      cmd_compare_recycling's per-row log for both recyclers.
  ref_hybrid.npz      HybridEvaluator (inversion.cpp:53-106) on a 33^2 experiment: K_* = 3
                      systems through the builder, then the reduced model.
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def desk_params(offset):
    """Desk::params (test_basis.cpp:43-52)."""
    p = np.zeros(16)
    for j in range(4):
        p[j] = 0.6 + offset
        p[4 + j] = 0.9
        p[8 + 2 * j] = 1.0 + 2.0 * (j % 2)
        p[8 + 2 * j + 1] = 1.0 + 2.0 * (j // 2)
    return p


def log_array(rows):
    return np.array([[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in rows])


def make_desk():
    n, ns, nd, k, tol = 21, 4, 4, 4, 1e-8
    offsets = [0.05, 0.1, 0.0, 0.3]
    g = ref.Grid(n, n)
    nodes = g.interior_nodes()
    pals = ref.Pals(m_bumps=4)
    src, det = ref.evenly_spaced_positions(n, ns), ref.evenly_spaced_positions(n, nd)
    B = g.layout(src, det)
    mu = lambda off: g.h ** 2 * pals.absorption(desk_params(off), nodes)  # noqa: E731
    mu0 = mu(0.0)
    out = dict(n=n, n_src=ns, n_det=nd, k=k, tol=tol, offsets=np.array(offsets), nodes=nodes, src=np.array(src),
               det=np.array(det), B=B, mu0=mu0, mus=np.stack([mu(o) for o in offsets]))
    # operator, MINRES
    x = np.random.default_rng(7).standard_normal(g.n)
    out["apply_x"], out["apply_y"] = x, g.apply(mu0, x)
    xs, rep = g.minres(mu0, B[:, 0], 1e-10, 2 * g.n)
    out["minres_x"], out["minres_hist"], out["minres_its"] = xs, rep.history, rep.iterations
    # seed
    rb = ref.Basis.init(g, mu0, B, k, tol)
    V = rb.V
    out["eigenvalues"], out["U0"], out["X0"] = rb.eigenvalues, V[:, :k].copy(), V[:, k:].copy()
    # per-RHS-only comparator from the same seed
    rec = ref.PerRhsRecycler(g, out["U0"], out["X0"])
    logs, psis, xnorm, cols, blogs = [], [], [], [], []
    Ct = B[:, ns:]
    for s, off in enumerate(offsets, start=1):
        pr = rb.process_system(mu(off), B, tol, s)
        logs.append(log_array(pr.log))
        psis.append(Ct.T @ pr.X[:, :ns])
        xnorm.append(np.linalg.norm(pr.X, axis=0))
        cols.append(rb.cols)
        pb = rec.solve_system(mu(off), B, tol, s)
        blogs.append(log_array(pb.log))
    out["log"], out["psi"], out["xnorm"], out["cols"] = np.concatenate(logs), np.stack(psis), np.stack(xnorm), np.array(cols)
    out["baseline_log"] = np.concatenate(blogs)
    out["markers"] = rb.markers
    out["spaces"] = np.array([len(rb.space(j)) for j in range(ns + nd)])
    Vf = rb.V
    out["R_diag_abs"] = np.abs(np.diag(rb.R))
    # recycled_minres on one raw space (columns of V and their images under system 2's operator)
    m2 = mu(offsets[1])
    W = Vf[:, : k + 3]
    AW = np.stack([g.apply(m2, W[:, j]) for j in range(W.shape[1])], axis=1)
    rhs = B[:, 1]
    corr, ndir, img, rrep = g.recycled_minres(m2, W, AW, rhs, 1e-9, 2 * g.n, float(np.linalg.norm(rhs)))
    out["rm_W"], out["rm_AW"], out["rm_corr"], out["rm_hist"], out["rm_its"] = W, AW, corr, rrep.history, rrep.iterations
    out["rm_corr_norm"] = rrep.correction_norm
    out["rm_z0"], out["rm_r0"] = ref.initial_guess(W, AW, rhs)  # initial_guess (krylov.cpp:141-145)
    # reduced model on the final basis at a new parameter
    rom = ref.ReducedModel(g, Vf)
    p_new = desk_params(0.17)
    mu_new = g.h ** 2 * pals.absorption(p_new, nodes)
    out["rom_mu"], out["rom_psi"] = mu_new, rom.transfer(mu_new)
    out["rom_jac"] = rom.jacobian(pals, p_new, nodes, g.h ** 2)
    out["pals_jac_cols"] = np.stack([pals.jacobian_column(p_new, kk, nodes) for kk in range(16)], axis=1)
    out["fom_psi"] = g.fom_transfer(mu_new)
    out["fom_jac"] = g.fom_jacobian(pals, p_new, nodes, g.h ** 2)
    out["V_final_shape"] = np.array(Vf.shape)
    np.savez_compressed(os.path.join(OUT, "ref_desk.npz"), **out)
    print("ref_desk: cols per system", cols, "iterations", [int(l[:, 3].sum()) for l in logs])


def make_criterion5():
    cfg = ref.exp_config(nx=121, ny=121, n_src=32, n_det=32, m_bumps=9, seed=1234)
    n, nrhs, npar = ref.exp_dims(cfg)
    with tempfile.TemporaryDirectory() as d:
        ours, base = ref.compare_recycling(cfg, d)
        rows = np.genfromtxt(os.path.join(d, "compare_recycling.csv"), delimiter=",", skip_header=1,
                             skip_footer=1)
    mus = []
    for i in range(3):
        mu, B = ref.exp_mu(cfg, i)
        mus.append(mu)
    out = dict(cfg=cfg, n=n, n_rhs=nrhs, params=np.stack([ref.exp_parameters(cfg, i) for i in range(3)]),
               mus=np.stack(mus), B_idx=np.argmax(np.abs(B), axis=0), B_val=B[np.argmax(np.abs(B), axis=0), np.arange(nrhs)],
               rows=rows, ours=ours, baseline=base, k_eig=10, tol=1e-7)
    np.savez_compressed(os.path.join(OUT, "ref_criterion5.npz"), **out)
    print("ref_criterion5: ours", ours, "baseline", base, "ratio", ours / base)


def make_hybrid():
    cfg = ref.exp_config(nx=33, ny=33, n_src=6, n_det=6, m_bumps=4, seed=11, k_systems=3, k_eig=6, tol_basis=1e-8)
    n, nrhs, npar = ref.exp_dims(cfg)
    ev = ref.HybridEvaluator(cfg)
    ps = [ref.exp_parameters(cfg, i) for i in range(6)]
    mus = [ref.exp_mu(cfg, i)[0] for i in range(6)]
    _, B = ref.exp_mu(cfg, 0)
    out = dict(cfg=cfg, n=n, n_rhs=nrhs, params=np.stack(ps), mus=np.stack(mus), B=B)
    out["psi0"] = ev.transfer(ps[0])
    V0 = ev.basis_V()
    out["U0"], out["X0"] = V0[:, :6].copy(), V0[:, 6: 6 + nrhs].copy()
    out["psi1"] = ev.transfer(ps[1])
    out["jac1"] = ev.jacobian(ps[1])
    out["psi2"] = ev.transfer(ps[2])
    out["psi3"] = ev.transfer(ps[3])
    st3 = ev.state()
    out["psi4_rom"] = ev.transfer(ps[4])  # K_* = 3 systems used: the reduced model
    out["jac4_rom"] = ev.jacobian(ps[4])
    st4 = ev.state()
    out["log"] = log_array(ev.build_log())
    out["state3"] = np.array([st3[k] for k in ("cols", "systems_used", "appends", "in_rom_mode", "full_order_solves")])
    out["state4"] = np.array([st4[k] for k in ("cols", "systems_used", "appends", "in_rom_mode", "full_order_solves")])
    # d mu / d p_k columns (absorption_jacobian) at p1 and p4 for the Jacobian contractions
    g = ref.Grid(33, 33)
    nodes = g.interior_nodes()
    pals = ref.Pals(m_bumps=4)
    out["dmu1"] = np.stack([pals.jacobian_column(ps[1], k, nodes) for k in range(npar)], axis=1)
    out["dmu4"] = np.stack([pals.jacobian_column(ps[4], k, nodes) for k in range(npar)], axis=1)
    out["h2"] = g.h ** 2
    try:
        ev.transfer(ps[0])  # p0 is not the cached point any more, and the ROM serves it
        ev_err = ""
    except ref.RefError as e:  # pragma: no cover
        ev_err = str(e)
    out["err"] = ev_err
    np.savez_compressed(os.path.join(OUT, "ref_hybrid.npz"), **out)
    print("ref_hybrid: state after 3 systems", st3, "after switch", st4)


if __name__ == "__main__":
    if not ref.available():
        raise SystemExit("oracle/_ref is not built and /root/reference is absent")
    which = sys.argv[1:] or ["desk", "criterion5", "hybrid"]
    for w in which:
        {"desk": make_desk, "criterion5": make_criterion5, "hybrid": make_hybrid}[w]()
