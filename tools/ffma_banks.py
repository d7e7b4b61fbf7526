"""Estimate register-bank (even/odd) conflicts of FFMAs in the hottest loop of a kernel."""
import re, subprocess, sys, collections
obj, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", sass):
    name = f.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    ins = [(int(m.group(1), 16), m.group(2).strip()) for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", f)]
    best = None
    for addr, txt in ins:
        mm = re.search(r"BRA.*?0x([0-9a-f]+)", txt)
        if mm and int(mm.group(1), 16) < addr:
            body = [t for a, t in ins if int(mm.group(1), 16) <= a <= addr]
            n = sum("FFMA" in t for t in body)
            if best is None or n > best[0]:
                best = (n, body)
    n, body = best
    conf = tot = 0
    for t in body:
        m = re.match(r"(?:@!?P\d\s+)?FFMA\s+R(\d+),\s*(-?R\d+)(\.reuse)?,\s*(-?R\d+)(\.reuse)?,\s*(-?R\d+)(\.reuse)?", t)
        if not m:
            continue
        tot += 1
        srcs = []
        for g in (2, 4, 6):
            r, reuse = m.group(g), m.group(g + 1)
            if not reuse:
                srcs.append(int(r.lstrip('-R')))
        par = collections.Counter(r % 2 for r in set(srcs))
        if max(par.values(), default=0) >= 2:
            conf += 1
    print(name[:100])
    print(f"loop FFMA {tot}, with >=2 same-parity non-reused sources: {conf} ({100*conf/max(tot,1):.1f}%)")
    print("instr in loop:", len(body), " non-FFMA:", len(body) - tot)
