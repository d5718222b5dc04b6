"""Per-kernel ms of the three inner projection kernels at C4 shape (n = 2M,
complex, c in a few recycle widths); optional env A/B via ROMDOT_* vars."""
import json, sys
sys.path.insert(0, '.')
from paper_1602_00138_b200 import romdot as R
CS = [int(a) for a in sys.argv[1:]] or [16, 40, 69, 81, 128]
for c in CS:
    ms = R.bench_projection(2097152, c, True, int(__import__('os').environ.get('PROJ_ITERS', '20')))
    es = 16; n = 2097152
    gb = [n * es * (c + e) / (m * 1e-3) / 1e9 for m, e in zip(ms, (1, 2, 9))]
    print(json.dumps({"c": c, "ms": [round(m, 4) for m in ms], "GBps": [round(g) for g in gb]}), flush=True)
