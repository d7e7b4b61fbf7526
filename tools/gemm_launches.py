"""List the distinct GEMM launches of one step from an ncu launch list: time, grid, template args.
Usage: gemm_launches.py launches.csv launches_per_step"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
L = [r for r in rows[hi + 1:] if len(r) > vi]
step = L[-int(sys.argv[2]):]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in step:
    m = re.search(r'gemm_kernel<(.*?)>', r[ki])
    if m:
        a = agg[(m.group(1), r[gi])]
        a[0] += 1
        a[1] += float(r[vi]) / 1e3
for (tmpl, grid), (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us / 1e3:8.3f} ms  n={n:3d}  {us / n:9.1f} us/launch  grid {grid:14s} <{tmpl}>")
