"""Sustained vs burst projection throughput with nvidia-smi sampling of SM /
memory clocks, power and throttle reasons (is the inner loop power-capped?)."""
import json, subprocess, sys, threading, time
sys.path.insert(0, '.')
from paper_1602_00138_b200 import romdot as R

rows = []
stop = False
def sampler():
    q = "clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active"
    while not stop:
        out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        rows.append((time.time(), out))
        time.sleep(0.05)

c = int(sys.argv[1]) if len(sys.argv) > 1 else 69
n = 2097152
for iters in (1, 3, 200):
    th = threading.Thread(target=sampler); stop = False; rows.clear(); th.start()
    t0 = time.time()
    ms = R.bench_projection(n, c, True, iters)
    stop = True; th.join()
    gb = [n * 16 * (c + e) / (m * 1e-3) / 1e9 for m, e in zip(ms, (1, 2, 9))]
    sm = sorted(int(r[1].split(",")[0]) for r in rows) if rows else [0]
    mem = sorted(int(r[1].split(",")[1]) for r in rows) if rows else [0]
    pw = sorted(float(r[1].split(",")[2]) for r in rows) if rows else [0]
    print(json.dumps({"iters": iters, "ms": [round(m, 4) for m in ms], "GBps": [round(g) for g in gb],
                      "sm_mhz_med": sm[len(sm) // 2], "mem_mhz_min": mem[0], "mem_mhz_med": mem[len(mem) // 2],
                      "power_w_max": pw[-1], "power_w_med": pw[len(pw) // 2],
                      "reasons": sorted(set(r[1].split(",")[3].strip() for r in rows)), "wall_s": round(time.time() - t0, 2)}),
          flush=True)
