"""Summarise an ncu --csv --metrics gpu__time_duration.sum launch list:
per kernel (template arguments shortened) launches, total ms, share, us/launch."""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*\)$", "", name)           # drop the parameter list
    name = name.replace("rd::", "")
    name = re.sub(r"\bdouble2\b", "double2", name)
    return name


def main(path, header=""):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r and "Metric Value" in r:
                hdr = {k: i for i, k in enumerate(r)}
            continue
        if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[hdr["Metric Unit"]]
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        k = short(r[hdr["Kernel Name"]])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    if header:
        print(header)
    print(f"{'kernel':62s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'us/launch':>10s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:62]:62s} {n:8d} {t / 1e3:10.2f} {100 * t / tot:6.1f}% {t / n:10.1f}")
    print(f"{'TOTAL':62s} {sum(n for n, _ in agg.values()):8d} {tot / 1e3:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
