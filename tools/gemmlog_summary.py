"""Aggregate the GEMMLOG lines of a dev_scale log by phase (sum over call sites and widths)."""
import re, sys, collections
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for line in open(sys.argv[1]):
    m = re.match(r'\s+([\d.]+) s\s+[\d.]+%\s+([\d.]+) TF/s n=\s*(\d+) .*?  (\S+)\|', line)
    if m:
        sec, tf, n, ph = float(m.group(1)), float(m.group(2)), int(m.group(3)), m.group(4)
        a = agg[ph]; a[0] += sec; a[1] += sec * tf; a[2] += n
tot = sum(a[0] for a in agg.values())
for ph, a in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f'{ph:16s} {a[0]:7.3f} s {100*a[0]/tot:5.1f}%  {a[1]/a[0]:6.2f} TF/s  launches {a[2]}')
print(f'listed total {tot:.3f} s')
