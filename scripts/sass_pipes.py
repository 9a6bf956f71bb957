"""Per-pipe instruction tally of a kernel from an ncu source-page CSV
(`ncu -i rep --page source --csv --print-source sass`): warp-level
instructions executed, grouped by the pipe the opcode issues to (the
B200 split: IADD3/LOP3/SEL/ISETP/... on ALU, IMAD/FFMA/... on FMA, MUFU/I2F
on XU).  Usage: sass_pipes.py src.csv [loop_count]"""
import csv
import re
import sys
from collections import Counter

ALU = {"IADD3", "LOP3", "SEL", "FSEL", "ISETP", "FSETP", "PLOP3", "SHF", "VIADD", "VIADDMNMX", "VIMNMX", "IMNMX",
       "PRMT", "P2R", "R2P", "LEA", "LOP", "FMNMX", "SHL", "SHR", "IABS", "BMSK", "SGXT", "LEA.HI", "IADD", "ISCADD",
       "VOTE", "VOTEU", "CS2R", "S2R", "FLO", "POPC", "BREV", "CCTL"}
FMA = {"IMAD", "FFMA", "FMUL", "FADD", "IMUL", "IADD32I", "MOV", "FFMA32I", "HFMA2", "IMAD32I", "FMUL32I"}
XU = {"MUFU", "I2F", "F2I", "F2F", "I2FP", "F2IP", "FRND"}


def pipe(op):
    base = op.split(".")[0]
    if base in XU:
        return "xu"
    if base in FMA:
        return "fma"
    if base in ALU:
        return "alu"
    return "other:" + base


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[1]
    src, ex = h.index("Source"), h.index("Instructions Executed")
    loops = float(sys.argv[2]) if len(sys.argv) > 2 else None
    c = Counter()
    ops = Counter()
    for r in rows[2:]:
        e = float(r[ex] or 0)
        if not e:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[src])
        if not m:
            continue
        op = m.group(2)
        p = pipe(op)
        c[p] += e
        ops[op.split(".")[0]] += e
    tot = sum(c.values())
    for k, v in c.most_common():
        print(f"{k:14s} {v:14.0f} {v / tot * 100:5.1f} %" + (f"  {v / loops:6.1f}/iter" if loops else ""))
    print("top opcodes:", ", ".join(f"{k} {v / (loops or tot):.1f}" for k, v in ops.most_common(25)))


if __name__ == "__main__":
    main()
