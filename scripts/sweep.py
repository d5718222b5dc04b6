"""C5 kernel sweep (BASELINE.json configs[4]) on the B200.

* stencil apply: 2D N in {317, 1000, 2000, 4000}, 3D N in {47, 100, 160, 252},
  D ~ U[0.3, 0.4], mu_a ~ U[0.005, 0.05] i.i.d. per node, real and complex;
  algorithmic bytes = ncols * n * 2 * es (x, y) + 32 n (assembled coefficients once).
* recycle-space projection kernels (TMA): n in {262144, 2097152}, k in
  {8, 32, 64, 128}; bytes per launch n*es*(k+1) / (k+2) / (k+9).
* RRQR: n in {262144, 2097152}, m in {64, 256, 1024}, A = Q diag(0.9^j) P;
  expected rank at 1e-10: 64 / 219 / 219.
Prints one JSON line per case; peak = MEASURED_PEAKS.json hbm_gbs.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import build, problem as P  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="stencil,proj,rrqr")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--ncols", default="1,4,8,16")
    args = ap.parse_args()
    build.build()
    from paper_1602_00138_b200 import romdot as R
    pk = peak()
    ctx = R.default_context()
    what = args.what.split(",")
    if "stencil" in what:
        cases = [(2, 317), (2, 1000), (2, 2000), (2, 4000), (3, 47), (3, 100), (3, 160), (3, 252)]
        if args.quick:
            cases = [(2, 1000), (3, 160)]
        for d, N in cases:
            g = P.GridSpec(d=d, N=(N,) * d, h=1.0 / (N - 1), D_bg=0.33)
            rng = np.random.default_rng(5)
            f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=0.0)
            for cplx in (False, True):
                dt = np.complex128 if cplx else np.float64
                op = R.SchurOperator(g, P.Fields(f.D, f.mu, g.h ** 2 * 0.1 if cplx else 0.0), dt)
                es = 16 if cplx else 8
                for ncols in [int(v) for v in args.ncols.split(",")]:
                    ms = R.bench_stencil(op, ncols, args.iters)
                    by = ncols * g.n * 2 * es + 32 * g.n
                    gbs = by / (ms * 1e-3) / 1e9
                    print(json.dumps({"kernel": "stencil", "d": d, "N": N, "n": g.n, "dtype": "c128" if cplx else "f64",
                                      "ncols": ncols, "ms": ms, "GBps": round(gbs, 1), "frac": round(gbs / pk, 3)}),
                          flush=True)
                del op
    if "refresh" in what:  # the C4 refresh shape: A_i W, 3D 128^3 complex, 96..768 columns
        g = P.CONFIGS["C4"].grid
        rng = np.random.default_rng(5)
        f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=g.h ** 2 * 0.1)
        op = R.SchurOperator(g, f, np.complex128)
        for ncols in (96, 256, 768):
            ms = R.bench_stencil(op, ncols, 3)
            by = ncols * g.n * 2 * 16 + 32 * g.n
            gbs = by / (ms * 1e-3) / 1e9
            print(json.dumps({"kernel": "stencil", "case": "C4 refresh A_i W", "d": 3, "N": 128, "n": g.n,
                              "dtype": "c128", "ncols": ncols, "ms": ms, "GBps": round(gbs, 1),
                              "frac": round(gbs / pk, 3)}), flush=True)
        del op
    if "proj" in what:
        for n in (262144, 2097152):
            for k in (8, 32, 64, 128):
                for cplx in (False, True):
                    es = 16 if cplx else 8
                    ms = R.bench_projection(n, k, cplx, args.iters)
                    for name, m, extra in (("T", ms[0], 1), ("NT", ms[1], 2), ("N+update", ms[2], 9)):
                        by = n * es * (k + extra)
                        gbs = by / (m * 1e-3) / 1e9
                        print(json.dumps({"kernel": f"ts_tma {name}", "n": n, "k": k, "dtype": "c128" if cplx else "f64",
                                          "ms": m, "GBps": round(gbs, 1), "frac": round(gbs / pk, 3)}), flush=True)
    if "rrqr" in what:
        import torch
        for n in (262144, 2097152):
            for m in (64, 256, 1024):
                if n * m * 8 > 20e9:
                    continue
                gen = torch.Generator(device="cuda").manual_seed(3)
                G = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=gen)
                Q, _ = torch.linalg.qr(G)
                del G
                scale = torch.tensor(0.9 ** np.arange(m), dtype=torch.float64, device="cuda")
                perm = torch.randperm(m, generator=torch.Generator().manual_seed(4)).cuda()
                A = (Q * scale)[:, perm].T.contiguous()  # (m, n) row-major == n x m column-major
                del Q
                torch.cuda.synchronize()
                import ctypes as C
                rank = C.c_long()
                pv = np.zeros(m, dtype=np.int64)
                rdg = np.zeros(m)
                t0 = time.perf_counter()
                R._check(R.load_library().rd_rrqr(ctx.h, 0, n, m, C.c_void_p(A.data_ptr()), 1e-10, 0, C.byref(rank),
                                                  R._p(pv), R._p(rdg), None, R.DEVICE))
                dt = time.perf_counter() - t0
                want = 64 if m == 64 else 219
                flops = 2.0 * n * m * m  # Householder-equivalent 2nm^2 - 2m^3/3, dominant term
                print(json.dumps({"kernel": "rrqr", "n": n, "m": m, "rank": rank.value, "expected_rank": want,
                                  "ok": rank.value == want, "s": round(dt, 4),
                                  "TFLOPs_equiv": round(flops / dt / 1e12, 2)}), flush=True)
                del A
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
