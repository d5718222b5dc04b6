"""Tall Gram throughput (TFLOP/s, real-flop count) at refresh / ROM / RRQR shapes."""
import json, sys
sys.path.insert(0, '.')
from paper_1602_00138_b200 import romdot as R
for (n, a, b, cplx, sym) in [(2097152, 768, 768, True, True), (2097152, 437, 437, True, True),
                             (2097152, 64, 64, True, True), (2097152, 768, 64, True, False),
                             (262144, 594, 594, False, True), (2097152, 1024, 1024, False, True)]:
    ms = R.bench_gram(n, a, b, cplx, sym, 3)
    fl = n * a * b * (8.0 if cplx else 2.0) * (0.5 if sym else 1.0)
    print(json.dumps({"n": n, "a": a, "b": b, "cplx": cplx, "sym": sym, "ms": round(ms, 3),
                      "TFLOPs": round(fl / (ms * 1e-3) / 1e12, 2)}), flush=True)
