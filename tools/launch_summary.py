"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py launches.csv [bench_steps]
"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    v = v / 1000 if r[ui] in ('nsecond', 'ns') else (v * 1000 if r[ui] in ('msecond', 'ms') else v)
    a = agg.setdefault(r[ki][:80], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"total {tot / steps:.1f} us per bench step, {sum(a[0] for a in agg.values()) / steps:.0f} launches")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / steps:9.1f} us {100 * t / tot:5.1f}% {c / steps:5.1f}x {t / c:8.1f} {n}")
