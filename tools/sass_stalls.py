"""Stall reasons per SASS opcode from an ncu --page source csv."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {n: i for i, n in enumerate(h)}
data = rows[2:]
cols = [c for c in h if c.startswith('stall_') and '(Not Issued)' not in c]
agg = collections.defaultdict(collections.Counter)
ex = collections.Counter()
for r in data:
    ins = r[1].strip().split()
    if not ins:
        continue
    o = (ins[1] if ins[0].startswith('@') else ins[0]).split('.')[0]
    for c in cols:
        try:
            agg[o][c] += float(r[idx[c]] or 0)
        except (ValueError, IndexError):
            pass
    try:
        ex[o] += float(r[idx['Instructions Executed']] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(sum(v.values()) for v in agg.values()) or 1
T = sum(ex.values()) or 1
print('instruction mix %:', {k: round(100 * v / T, 1) for k, v in ex.most_common(10)})
for o, _ in ex.most_common(6):
    print(f'stalls at {o:8s}', {k.replace('stall_', ''): round(100 * v / tot, 1) for k, v in agg[o].most_common(5)})
