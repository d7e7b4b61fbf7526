"""Per-function SASS opcode counts grouped by issue pipe (B300_MICROARCH.md 'Pipe rates':
IMAD/FFMA/FMUL on the FMA pipe, IADD3/LOP3/SHF/PRMT/... on the ALU pipe).
Usage: sass_pipes.py <cubin|so> <function-regex>"""
import collections, re, subprocess, sys

FMA = {"IMAD", "FFMA", "FMUL", "FADD", "FFMA2", "FMUL2", "FADD2", "HFMA2", "IMUL"}
ALU = {"IADD3", "LOP3", "SHF", "PRMT", "FMNMX", "ISETP", "SEL", "LEA", "IADD", "VIADD", "MOV", "IABS", "FSETP",
       "PLOP3", "FSEL", "LOP", "SHL", "SHR", "BMSK"}
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", sass)[1:]:
    name = f.split("\n", 1)[0].strip()
    if not re.search(sys.argv[2], name):
        continue
    ops = collections.Counter(re.findall(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", f, re.M))
    fma = sum(v for k, v in ops.items() if k in FMA)
    alu = sum(v for k, v in ops.items() if k in ALU)
    tot = sum(ops.values())
    print(f"{name[:90]}\n  total {tot}  fma-pipe {fma}  alu-pipe {alu}  other {tot - fma - alu}")
    print("  " + " ".join(f"{k}:{v}" for k, v in ops.most_common(12)))
