"""Kernel-time shares (and DRAM traffic) of one step from an ncu launch list
(--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv).
Usage: launch_shares.py launches.csv launches_per_step [marker_kernel step_index]
  (with a marker: the step = the launches from the step_index-th launch of marker_kernel
   up to the next one)"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ii, ki, mi, vi = h.index('ID'), h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[ii], {'name': r[ki]})
    d[r[mi]] = float(r[vi].replace(',', ''))
per = int(sys.argv[2])
allv = list(launch.values())
if len(sys.argv) > 4:
    marks = [i for i, d in enumerate(allv) if sys.argv[3] in d['name']]
    k = int(sys.argv[4])
    step = allv[marks[k]:marks[k + 1]]
    assert per == 0 or len(step) == per, (len(step), per)
else:
    step = allv[-per:]


def short(k):
    k = k.replace('(anonymous namespace)::', '').replace('<unnamed>::', '')
    m = re.search(r'gemm_kernel<(\d+), (\d+)(?:, \d+)+, (true|false|0|1), (true|false|0|1), (\d), (true|false|0|1)', k)
    if m:
        t = lambda x: 'T' if x in ('true', '1') else 'N'  # noqa: E731
        return 'gemm_kernel %sx%s %s%s%s' % (m.group(1), m.group(2), t(m.group(3)), t(m.group(4)),
                                            ' XP' if t(m.group(6)) == 'T' and t(m.group(3)) == 'N' else '')
    m = re.search(r'gemm_tn_kernel<(\d+), (\d+)', k)
    if m:
        return 'gemm_tn_kernel %sx%s TN (gemm_tn.cu)' % (m.group(1), m.group(2))
    return re.sub(r'\(.*', '', k).replace('void ', '')


tot, cnt, byt = collections.defaultdict(float), collections.Counter(), collections.defaultdict(float)
for d in step:
    k = short(d['name'])
    tot[k] += d.get('gpu__time_duration.sum', 0.0)
    byt[k] += d.get('dram__bytes_read.sum', 0.0) + d.get('dram__bytes_write.sum', 0.0)
    cnt[k] += 1
T = sum(tot.values())
B = sum(byt.values())
print(f"launches in the step: {len(step)}; serialized kernel time {T / 1e6:.2f} ms; DRAM traffic {B / 1e9:.2f} GB "
      "(ncu replay: cold cache, serialized, --clock-control none)")
print(f"{'ms':>9s} {'share':>6s} {'n':>5s} {'GB':>8s} {'GB/s':>7s}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    gbs = byt[k] / v if v else 0.0  # bytes / ns = GB/s
    print(f"{v / 1e6:9.3f} {100 * v / T:5.1f}% {cnt[k]:5d} {byt[k] / 1e9:8.3f} {gbs:7.0f}  {k}")
