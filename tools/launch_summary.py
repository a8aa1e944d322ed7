"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name: count, total, share."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        v = float(r[mi].replace(",", ""))
        unit = r[ui] if ui is not None else "ns"
        v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = ["%-40s %6s %12s %10s %7s" % ("kernel", "n", "total_us", "avg_us", "share")]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append("%-40s %6d %12.1f %10.2f %6.1f%%" % (k, n, t, t / n, 100 * t / tot))
    out.append("total_us %.1f launches %d" % (tot, sum(v[0] for v in agg.values())))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
