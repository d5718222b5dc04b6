"""RRQR at the C5 shape (n = 2,097,152, m = 1024, decay 0.9): cold and warm call times; PROF=1
brackets the warm call with cudaProfilerStart/Stop for ncu --profile-from-start off."""
import ctypes as C, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_1602_00138_b200 import romdot as R
n, m = int(os.environ.get("RN", 2097152)), int(os.environ.get("RM", 1024))
ctx = R.default_context()
gen = torch.Generator(device="cuda").manual_seed(3)
G = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=gen)
Q, _ = torch.linalg.qr(G); del G
scale = torch.tensor(0.9 ** np.arange(m), dtype=torch.float64, device="cuda")
perm = torch.randperm(m, generator=torch.Generator().manual_seed(4)).cuda()
A = (Q * scale)[:, perm].T.contiguous(); del Q
torch.cuda.synchronize()
for rep in range(3):
    rank = C.c_long(); pv = np.zeros(m, dtype=np.int64); rdg = np.zeros(m)
    if rep == 2 and os.environ.get("PROF"):
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    R._check(R.load_library().rd_rrqr(ctx.h, 0, n, m, C.c_void_p(A.data_ptr()), 1e-10, 0, C.byref(rank), R._p(pv), R._p(rdg), None, R.DEVICE))
    dt = time.perf_counter() - t0
    if rep == 2 and os.environ.get("PROF"):
        torch.cuda.profiler.stop()
    print(f"call {rep}: {dt*1e3:.1f} ms rank {rank.value} TFLOPs-equivalent {2.0*n*m*m/dt/1e12:.2f}", flush=True)
