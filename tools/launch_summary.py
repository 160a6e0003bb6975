"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches,
total time and share (cold-cache, serialised: compare shares, not absolutes)."""
import csv
import sys
from collections import defaultdict


def main(path, header=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "ns"
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        tot[r[ki]] += ms
        cnt[r[ki]] += 1
    allms = sum(tot.values())
    if header:
        print(header)
    print("(cold-cache, serialised per-launch times; compare shares, not absolutes)")
    print("launches      total_ms  share  kernel")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print("%8d  %12.2f  %4.1f%%  %s" % (cnt[k], tot[k], 100 * tot[k] / allms, k[:72]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
