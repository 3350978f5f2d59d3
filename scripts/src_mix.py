"""Instruction mix of each kernel in an ncu source CSV (executed warp
instructions by SASS opcode), to see where a pass's issue slots go."""
import csv, gzip, io, sys
from collections import Counter

data = (gzip.open if sys.argv[1].endswith(".gz") else open)(sys.argv[1], "rt").read()
seen = set()
for blk in data.split('"Kernel Name",')[1:]:
    name, rest = blk.split("\n", 1)
    if name in seen:
        continue
    seen.add(name)
    rows = list(csv.reader(io.StringIO(rest)))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    c = Counter()
    tot = 0
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        n = int(r[ix["Instructions Executed"]] or 0)
        src = r[ix["Source"]].strip()
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        op = op.split(".")[0]
        c[op] += n
        tot += n
    print(name[:150], "total warp-instr", tot)
    print("  " + ", ".join(f"{k}={v/tot:.1%}" for k, v in c.most_common(28)))
