"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total device ms, share. Usage: python tools/launch_summary.py launches.csv [out.csv]"""

import csv
import re
import sys
from collections import OrderedDict


def main():
    src = sys.argv[1]
    rows = []
    with open(src) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        rows.append((name, ms))
    agg = OrderedDict()
    for name, ms in rows:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    out = sorted(agg.items(), key=lambda kv: -kv[1][1])
    w = csv.writer(open(sys.argv[2], "w", newline="")) if len(sys.argv) > 2 else None
    if w:
        w.writerow(["kernel", "launches", "device_ms", "share"])
    for name, (cnt, ms) in out:
        print(f"{name[:90]:90s} {cnt:6d} {ms:10.3f} ms {100 * ms / tot:6.2f}%")
        if w:
            w.writerow([name, cnt, f"{ms:.4f}", f"{ms / tot:.4f}"])
    print(f"total {len(rows)} launches, {tot:.2f} ms")


if __name__ == "__main__":
    main()
