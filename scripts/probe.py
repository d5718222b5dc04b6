"""Kernel probe for ncu / timing: one recycled CG/COCG solve of fixed length on
a BASELINE config's operator with a recycle space of width c (device buffers),
plus standalone stencil applies. Usage:
  python scripts/probe.py --config C4 --width 80 --iters 20
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1602_00138_b200 import build, problem as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--width", type=int, default=48)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--stencil-cols", type=int, default=8)
    ap.add_argument("--no-events", action="store_true", help="no per-launch CUDA events (wall time per iteration only)")
    args = ap.parse_args()
    import torch
    build.build()
    from paper_1602_00138_b200 import romdot as R
    cfg = P.CONFIGS[args.config]
    g, lay = cfg.grid, cfg.layout()
    n = g.n
    dt = np.dtype(cfg.dtype)
    tdt = torch.complex128 if cfg.complex else torch.float64
    ctx = R.Context(0)
    f = cfg.fields(1, cfg.omegas[-1])
    op = R.SchurOperator(g, f, dt, ctx)
    c = args.width
    gen = torch.Generator(device="cuda").manual_seed(0)
    U = torch.randn((c, n), dtype=tdt, device="cuda", generator=gen)
    K = torch.randn((c, n), dtype=tdt, device="cuda", generator=gen)
    K /= K.norm(dim=1, keepdim=True)
    rhs = torch.zeros(n, dtype=tdt, device="cuda")
    rhs[int(lay.idx[0])] = lay.val[0]
    outs = [torch.empty(n, dtype=tdt, device="cuda") for _ in range(3)]
    rep = R._Report()
    L = R.load_library()
    ctx.profile(not args.no_events)
    for r in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        R._check(L.rd_recycled_solve(op.h, R._dt(dt), U.data_ptr(), K.data_ptr(), c, rhs.data_ptr(), 1e-30,
                                     args.iters, abs(lay.val[0]), outs[0].data_ptr(), outs[1].data_ptr(),
                                     outs[2].data_ptr(), C.byref(rep), None, 0, R.DEVICE))
        torch.cuda.synchronize()
        print(f"solve rep {r}: {rep.iterations} its, relres {rep.final_relres:.6e}, {(time.perf_counter() - t0) * 1e3 / max(1, rep.iterations):.3f} ms/it")
    for k, (ms, by, ns) in ctx.prof().items():
        if ns:
            print(f"  {k:16s} {ms / ns * 1e3:9.1f} us/launch  {by / (ms / 1e3) / 1e9:8.1f} GB/s  ({ns} samples)")
    X = torch.randn((args.stencil_cols, n), dtype=tdt, device="cuda", generator=gen)
    Y = torch.empty_like(X)
    for r in range(args.reps):
        torch.cuda.synchronize()
        ctx.mark()
        R._check(L.rd_op_apply(op.h, R._dt(dt), X.data_ptr(), Y.data_ptr(), args.stencil_cols, R.DEVICE))
        ctx.mark()
        ms = ctx.elapsed_ms()
        es = dt.itemsize
        by = args.stencil_cols * n * 2 * es + n * 4 * 8
        print(f"stencil x{args.stencil_cols}: {ms:.3f} ms, {by / (ms / 1e3) / 1e9:.1f} GB/s (alg. bytes incl. 4 coeff fields once)")


if __name__ == "__main__":
    main()
