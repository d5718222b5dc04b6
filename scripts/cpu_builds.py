"""CPU-checker full basis builds for the BASELINE.md table (C1 .. C3), timed on
the host cores of the box it runs on: checker seed (shift-invert Lanczos +
X0 solves) + every system (process_system, proj/src/basis.cpp:157-207) +
QRCP at 1e-10. One JSON line per (config, threads).

  python scripts/cpu_builds.py --configs C1,C3 --threads 1,16
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(cfg_name: str, systems: int) -> dict:
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    from paper_1602_00138_b200 import problem as P
    c = P.CONFIGS[cfg_name]
    g, lay = c.grid, c.layout()
    t0 = time.perf_counter()
    f0 = c.fields(0)
    _, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, min(c.tol, 1e-8))
    X0, x0_its = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    t_seed = time.perf_counter() - t0
    gb = orc.GlobalBasis(U0.astype(c.dtype), X0, c.cap)
    solves = its = 0
    per = []
    syst = c.systems()[:systems] if systems else c.systems()
    for s, (pt, w) in enumerate(syst, start=1):
        t1 = time.perf_counter()
        po = orc.process_system(gb, orc.Operator.grid(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
        per.append(round(time.perf_counter() - t1, 2))
        solves += sum(1 for r in po.log if r.iterations > 0)
        its += po.inner_iterations
    t2 = time.perf_counter()
    rank, _, _, _ = orc.qrcp(gb.V, 1e-10, True)
    t_qr = time.perf_counter() - t2
    total = time.perf_counter() - t0
    return {"config": cfg_name, "threads": int(os.environ.get("OMP_NUM_THREADS", "0")), "systems": len(syst),
            "basis_build_s": round(total, 2), "seed_s": round(t_seed, 2), "systems_s": per,
            "qrcp_s": round(t_qr, 2), "solves": solves, "inner_iterations": its, "rank": int(rank),
            "solves_per_s": round(solves / max(1e-9, sum(per)), 4), "host_cores": os.cpu_count()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C3")
    ap.add_argument("--threads", default="1,16")
    ap.add_argument("--systems", type=int, default=0)
    ap.add_argument("--child", default="")
    args = ap.parse_args()
    if args.child:
        print(json.dumps(one(args.child, args.systems)), flush=True)
        return
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    for cfg in args.configs.split(","):
        for th in args.threads.split(","):
            env = dict(os.environ, OMP_NUM_THREADS=th)
            subprocess.run([sys.executable, __file__, "--child", cfg, "--systems", str(args.systems)], env=env)


if __name__ == "__main__":
    main()
