"""Kernel-time shares of one step from an ncu launch list (gpu__time_duration.sum csv).
Usage: launch_shares.py launches.csv n_steps_profiled"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
ts = [(r[ki], float(r[vi])) for r in rows[hi + 1:] if len(r) > vi]
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
# take the last 1/nsteps of the launches as one step
step = ts[len(ts) - len(ts) // nsteps:]
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, v in step:
    k = k.replace('(anonymous namespace)::', '').replace('<unnamed>::', '')
    m = re.search(r'gemm_kernel<(\d+), (\d+)(?:, \d+)+, (true|false|0|1), (true|false|0|1)', k)
    if m:
        k = 'gemm_kernel %sx%s %s%s' % (m.group(1), m.group(2), 'T' if m.group(3) in ('true', '1') else 'N',
                                        'T' if m.group(4) in ('true', '1') else 'N')
    else:
        k = re.sub(r'\(.*', '', k).replace('void ', '')
    tot[k] += v
    cnt[k] += 1
T = sum(tot.values())
print(f"launches in the step: {len(step)}; serialized kernel time {T / 1e6:.2f} ms (cold-cache ncu replay)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6:9.3f} ms {100 * v / T:5.1f}%  n={cnt[k]:4d}  {k}")
