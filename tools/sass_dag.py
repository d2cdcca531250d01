#!/usr/bin/env python
"""Critical path of a SASS address range (straight-line; register and
predicate true dependencies only) under assumed latencies, next to the
compiler's static schedule (sum of stall counts) for the same range.

    python tools/sass_dag.py <file.sass> <lo_hex> <hi_hex>
"""
import re
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from sass_sched import parse  # noqa: E402

LAT = {"DADD": 8, "DMUL": 8, "DFMA": 8, "DSETP": 8, "MUFU": 20, "SHFL": 24, "LDS": 30, "LDL": 30}
WIDE = ("DADD", "DMUL", "DFMA", "DSETP", "MUFU.RSQ64H", "MUFU.RCP64H")


def regs(tok, wide):
    out = []
    for m in re.finditer(r'(-|\|)?\b(R\d+|P\d+|UR\d+)\b', tok):
        r = m.group(2)
        if r in ("RZ", "PT"):
            continue
        out.append(r)
        if wide and r.startswith("R"):
            out.append("R%d" % (int(r[1:]) + 1))
    return out


def analyse(ins):
    ready = {}
    crit = 0
    for a, t, c in ins:
        t2 = re.sub(r'^@!?\w+\s+', '', t)
        op = t2.split()[0]
        base = op.split('.')[0]
        args = t2[len(op):].split(',')
        wide = base in ("DADD", "DMUL", "DFMA") or op.startswith("MUFU.RSQ64H")
        pred_pos = base in ("DSETP", "ISETP", "FSETP", "PLOP3")
        if base in ("DSETP", "ISETP", "FSETP", "PLOP3", "LOP3") and re.match(r'\s*P\d', args[0] if args else ''):
            dst, src = regs(args[0], False) + (regs(args[1], False) if len(args) > 1 and re.match(r'\s*P\d', args[1]) else []), args[1:]
        else:
            dst, src = (regs(args[0], wide and not op.startswith("MUFU")) if args else []), args[1:]
        if op.startswith("MUFU.RSQ64H"):
            dst = regs(args[0], False)
        srcs = []
        gp = re.match(r'^@!?(\w+)', t)
        if gp:
            srcs.append(gp.group(1))
        for s in src:
            w = base in ("DADD", "DMUL", "DFMA", "DSETP")
            srcs += regs(s, w and not re.search(r'\bP\d', s))
        start = max([ready.get(r, 0) for r in srcs] + [0])
        lat = LAT.get(base, 4)
        for r in dst:
            ready[r] = start + lat
        crit = max(crit, start + lat)
    return crit


def main():
    path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
    ins = [x for x in parse(path) if lo <= x[0] <= hi]
    stall = sum(c & 0xF for _, _, c in ins)
    print(f"instructions {len(ins)}  static schedule {stall}  critical path {analyse(ins)}")


if __name__ == "__main__":
    main()
