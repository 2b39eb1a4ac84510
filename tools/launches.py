"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel.

usage: python tools/launches.py launches.csv [--from-id N]
"""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    iname, ival, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    out = []
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        v = float(r[ival].replace(",", ""))
        unit = r[unit_i] if unit_i is not None else "nsecond"
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        out.append((int(r[iid]), r[iname], v * scale))
    return out


def summarise(data, title=""):
    agg = collections.OrderedDict()
    for _, nm, us in data:
        short = nm.split("(")[0]
        short = short.replace("skel::<unnamed>::", "")[:70]
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(us for _, _, us in data)
    lines = [f"# {title} total {tot:.1f} us over {len(data)} launches"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v:10.1f} us {c:5d}x {100 * v / tot:5.1f}%  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    d = load(sys.argv[1])
    start = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--from-id" else len(d) // 2
    print(summarise(d[start:], sys.argv[1]))
