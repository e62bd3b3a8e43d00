"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count, time, share."""
import csv
import sys
from collections import defaultdict


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
        unit = r[ui]
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3}.get(unit, 1.0)
    total = sum(tot.values())
    lines = [f"{'kernel':58s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>7s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{k[:58]:58s} {cnt[k]:8d} {tot[k] * scale:10.3f} {tot[k] * scale / cnt[k]:9.3f} "
                     f"{100 * tot[k] / total:6.2f}%")
    lines.append(f"{'total':58s} {sum(cnt.values()):8d} {total * scale:10.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
