"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into one bench step.
usage: python tools/launch_summary.py profiles/round1/launches_c2k512.csv > profiles/round1/launches_c2k512_step.txt"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith('==')]
rows = list(csv.reader(lines))
hdr = rows[0]
iname, ival = hdr.index('Kernel Name'), hdr.index('Metric Value')
data = [(r[iname].split('(')[0].replace('void ', '').replace('skel::<unnamed>::', ''), float(r[ival]) / 1000)
        for r in rows[1:] if len(r) == len(hdr)]
starts = [i for i, (n, t) in enumerate(data) if 'k_omega_image' in n]
seg = data[starts[-2]:starts[-1]] if len(starts) > 1 else data[starts[-1]:]
agg = collections.OrderedDict()
for n, t in seg:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(t for _, t in seg)
sel = []
for n, t in seg:
    if 'k_cpqr' in n:
        break
    sel.append((n, t))
stot = sum(t for _, t in sel)
sk = sum(t for n, t in sel if 'omega' in n or 'sketch' in n)
print(f"# one bench.py step (C2 k=512): {len(seg)} launches, {tot:.1f} us (ncu, serialized, cold caches)")
print(f"# selection (sketch + column LUPP) = first {len(sel)} launches, {stot:.1f} us; sketch kernels {sk:.1f} us = "
      f"{100 * sk / stot:.1f}% of it")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us {c:4d}x {100 * t / tot:5.1f}%  {n}")
