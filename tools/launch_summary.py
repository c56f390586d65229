"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, out, title):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ik, iu, iv = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    tot = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        us = float(r[iv].replace(",", "")) * SCALE[r[iu]]
        name = r[ik].split("(")[0]
        c, s = tot.get(name, (0, 0.0))
        tot[name] = (c + 1, s + us)
    allt = sum(s for _, s in tot.values())
    lines = [title, "per-launch times are cold-cache and serialised; compare SHARES, not absolutes", "",
             f"{'kernel':64s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>6s}"]
    for name, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:64]:64s} {c:8d} {s:11.1f} {s / c:9.2f} {100 * s / allt:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])
