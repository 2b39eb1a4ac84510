"""Per-kernel table of an ncu launch list (gpu__time_duration.sum per launch) of one bench.py step:
count, total device time and share of this library's kernels (names in skel's anonymous namespace
or k_*; library GEMMs other processes launch, e.g. torch building the input, are listed apart).
usage: python tools/launch_table.py gpurun_out/launches.csv [title] > profiles/roundN/launches_<cfg>.txt"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith('==')]
rows = list(csv.reader(lines))
hdr = rows[0]
iname, ival, iunit = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6, 's': 1e6}
ours, other = collections.OrderedDict(), collections.OrderedDict()
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    raw = r[iname]
    name = raw.split('(')[0].replace('void ', '').replace('skel::<unnamed>::', '').replace('unnamed>::', '')
    us = float(r[ival]) * scale.get(r[iunit], 1.0)
    mine = 'unnamed>' in raw or name.startswith('k_') or 'skel::' in raw
    a = (ours if mine else other).setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(v[1] for v in ours.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print(f"# library kernels: {sum(v[0] for v in ours.values())} launches, {tot / 1e3:.2f} ms (ncu: serialised, cold caches "
      f"-- compare shares, not absolutes)")
for name, (cnt, us) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
    print(f"{us / 1e3:12.3f} ms {cnt:6d}x {100 * us / tot:6.2f}%  {name}")
if other:
    print(f"# other launches in the process (input construction etc.): {sum(v[0] for v in other.values())}, "
          f"{sum(v[1] for v in other.values()) / 1e3:.2f} ms")
