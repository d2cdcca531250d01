#!/usr/bin/env python
"""Static schedule of a SASS address range from cuobjdump -sass output:
decodes the Volta+ control bits of every instruction (stall cycles, yield,
write / read scoreboard, wait mask) and sums the stall counts — the
compiler's own fixed-latency issue schedule for that range (variable-latency
waits on scoreboards, e.g. MUFU / LDS / shuffles, come on top).

    python tools/sass_sched.py <file.sass> <lo_hex> <hi_hex> [--list]
"""
import re
import sys
from collections import Counter


def parse(path):
    lines = open(path).read().splitlines()
    out = []
    i = 0
    while i < len(lines):
        m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?)\s*;\s*/\* (0x[0-9a-f]+) \*/', lines[i])
        if m:
            hi = re.search(r'/\* (0x[0-9a-f]+) \*/', lines[i + 1])
            ctrl = (int(hi.group(1), 16) >> 41) & 0x1FFFF if hi else 0
            out.append((int(m.group(1), 16), m.group(2), ctrl))
            i += 2
        else:
            i += 1
    return out


def main():
    path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
    ins = [x for x in parse(path) if lo <= x[0] <= hi]
    cyc = 0
    ops = Counter()
    waits = 0
    for a, t, c in ins:
        stall, yld, wb, rb, wm = c & 0xF, (c >> 4) & 1, (c >> 5) & 7, (c >> 8) & 7, (c >> 11) & 0x3F
        cyc += stall
        op = t.split()[0]
        if op.startswith('@'):
            op = t.split()[1]
        ops[op.split('.')[0]] += 1
        waits += wm != 0
        if '--list' in sys.argv:
            print(f"{a:05x} s{stall:2d} wb{wb if wb != 7 else '-'} rb{rb if rb != 7 else '-'} "
                  f"w{wm:06b} {t}")
    fp64 = sum(v for k, v in ops.items() if k in ('DADD', 'DMUL', 'DFMA', 'DSETP', 'DMNMX'))
    print(f"instructions {len(ins)}  fp64 {fp64}  stall-cycle sum {cyc}  scoreboard waits {waits}")
    print(sorted(ops.items(), key=lambda x: -x[1])[:20])


if __name__ == "__main__":
    main()
