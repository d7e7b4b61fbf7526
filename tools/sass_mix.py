"""Instruction mix of the hottest loop of a kernel in a cubin/.o (SASS)."""
import re, subprocess, sys, collections
obj, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs:
    name = f.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    # find backward branches -> loops
    best = None
    for addr, txt in ins:
        m = re.match(r"(@!?U?P\d+\s+)?BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
        mm = re.search(r"BRA.*?0x([0-9a-f]+)", txt)
        if mm:
            tgt = int(mm.group(1), 16)
            if tgt < addr:
                body = [t for a, t in ins if tgt <= a <= addr]
                nffma = sum(1 for t in body if "FFMA" in t)
                if best is None or nffma > best[0]:
                    best = (nffma, tgt, addr, body)
    print("==", name[:120])
    if best:
        nffma, tgt, addr, body = best
        c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
        print(f"loop {tgt:#x}-{addr:#x}: {len(body)} instr, FFMA {nffma} ({100*nffma/len(body):.1f}%)")
        print(dict(c.most_common(12)))
        reuse = sum(1 for t in body if "FFMA" in t and ".reuse" in t)
        print("FFMA with reuse:", reuse)
