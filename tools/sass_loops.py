"""Summarise the loops (backward branches) of one SASS function: instruction
mix per loop body. usage: sass_loops.py <sass file> <function substring>"""
import re
import sys
from collections import Counter

text = open(sys.argv[1]).read()
funcs = re.split(r"\n\s*Function : ", text)
body = next(f for f in funcs if sys.argv[2] in f.split("\n", 1)[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:`\()?(?:\.L_x_\d+|0x([0-9a-f]+))", txt)
    mt = re.search(r"0x([0-9a-f]+)", txt) if "BRA" in txt else None
    if "BRA" in txt and mt:
        tgt = int(mt.group(1), 16)
        if tgt < a and tgt in addr_idx:
            loop = ins[addr_idx[tgt]:i + 1]
            c = Counter()
            for _, t in loop:
                op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
                c[op.split(".")[0]] += 1
            fp64 = sum(c[k] for k in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX"))
            print(f"loop 0x{tgt:x}-0x{a:x}: {len(loop)} instr, fp64={fp64}, "
                  + ", ".join(f"{k}:{v}" for k, v in c.most_common(14)))
