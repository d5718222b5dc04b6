"""One-paragraph summary of an `ncu --set full` capture exported with
`ncu -i X.ncu-rep --page raw --csv > X_raw.csv`: duration, DRAM traffic and
throughput, L2 hit rate, FP64 / tensor-pipe (DMMA) utilisation, occupancy.
  python scripts/ncu_raw_summary.py profiles/r02_gram_c128_768_raw.csv [alg_bytes] [flops]
"""
import csv
import sys

KEYS = {
    "name": "Kernel Name",
    "t_ms": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "dmma_inst_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "tensor_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "fp64_inst_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "fp64_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem": "launch__shared_mem_per_block_dynamic",
    "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1.0, "us": 1e-3, "ns": 1e-6,
         "s": 1e3, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "Ghz": 1e3, "Mhz": 1.0, "hz": 1e-6,
         "cycle/second": 1e-6, "cycle/nsecond": 1e3, "cycle/usecond": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {}
        for k, col in KEYS.items():
            if col in hdr:
                i = hdr.index(col)
                v, u = vals[i], units[i]
                if k == "name":
                    d[k] = v
                    continue
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                d[k] = x * SCALE.get(u.split("/")[0] if k == "smem" else u, 1.0) \
                    if k in ("dram_rd", "dram_wr", "t_ms", "sm_mhz", "smem") else x
        out.append(d)
    return out


def main():
    path = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    flops = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    for d in load(path):
        t = d.get("t_ms", 0.0)
        tr = d.get("dram_rd", 0.0) + d.get("dram_wr", 0.0)
        s = [f"{d.get('name', '?')[:90]}",
             f"duration {t:.3f} ms, grid {int(d.get('grid', 0))} x {int(d.get('block', 0))}, "
             f"{int(d.get('regs', 0))} regs, dyn smem {d.get('smem', 0) / 1e3:.0f} KB, SM clock {d.get('sm_mhz', 0):.0f} MHz",
             f"DRAM read {d.get('dram_rd', 0) / 1e9:.3f} GB + write {d.get('dram_wr', 0) / 1e9:.3f} GB = "
             f"{tr / 1e9:.3f} GB ({tr / (t * 1e-3) / 1e9 if t else 0:.0f} GB/s), "
             f"DRAM throughput {d.get('dram_pct', 0):.1f}% of ncu peak, L2 hit {d.get('l2_hit', 0):.1f}%",
             f"SM throughput {d.get('sm_pct', 0):.1f}%, warps active {d.get('occ', 0):.1f}%, "
             f"DMMA inst {d.get('dmma_inst_pct', 0):.1f}% of peak, tensor pipe active {d.get('tensor_active_pct', 0):.1f}%, "
             f"FP64 (DFMA) pipe {d.get('fp64_inst_pct', 0):.1f}%"]
        if alg:
            s.append(f"algorithmic bytes {alg / 1e9:.3f} GB -> {alg / (t * 1e-3) / 1e9:.0f} GB/s; "
                     f"traffic / algorithmic = {tr / alg:.3f}")
        if flops:
            s.append(f"{flops / 1e12:.3f} TFLOP -> {flops / (t * 1e-3) / 1e12:.2f} TFLOP/s")
        print("\n".join(s))


if __name__ == "__main__":
    main()
