"""Per-opcode executed instructions and warp-stall samples of one kernel from
`ncu -i REP --page source --csv --print-source sass` output (stdin or file)."""
import csv
import sys
from collections import Counter


def sections(path):
    rows = list(csv.reader(open(path)))
    cur, name, hdr = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            if name:
                yield name, hdr, cur
            name, hdr, cur = r[1], None, []
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and len(r) == len(hdr):
            cur.append(r)
    if name:
        yield name, hdr, cur


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


for name, hdr, data in sections(sys.argv[1]):
    if len(sys.argv) > 2 and sys.argv[2] not in name:
        continue
    i_src, i_all, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot_s = sum(num(r[i_all]) for r in data)
    tot_e = sum(num(r[i_ex]) for r in data)
    c, cs = Counter(), Counter()
    for r in data:
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        c[op] += num(r[i_ex])
        cs[op] += num(r[i_all])
    print(f"== {name}: {len(data)} SASS instr, {tot_e:.3e} warp-instr executed, {tot_s:.0f} stall samples")
    for k, v in c.most_common(22):
        print(f"   {k:10s} {v / tot_e * 100:6.2f}% of executed   {cs[k] / tot_s * 100:6.2f}% of stall samples")
