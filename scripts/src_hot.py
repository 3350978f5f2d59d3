"""Summarise an ncu --page source --csv --print-source sass dump: per kernel,
the stall-sample totals by reason and the hottest instructions (with their
shared-memory excess wavefronts)."""
import csv, gzip, io, sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
data = (gzip.open if path.endswith(".gz") else open)(path, "rt").read()
blocks = data.split('"Kernel Name",')[1:]
for blk in blocks:
    name, rest = blk.split("\n", 1)
    rows = list(csv.reader(io.StringIO(rest)))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    body = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
    print("=" * 100)
    print(name[:160], "samples", tot)
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    c = Counter()
    for r in body:
        for k in stalls:
            c[k] += int(r[ix[k]] or 0)
    print("  stall totals:", ", ".join(f"{k[6:]}={v/tot:.1%}" for k, v in c.most_common(10)))
    exc = sum(int(r[ix["L1 Wavefronts Shared Excessive"]] or 0) for r in body)
    wf = sum(int(r[ix["L1 Wavefronts Shared"]] or 0) for r in body)
    print(f"  shared wavefronts {wf}, excessive {exc}")
    body.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for r in body[:top]:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        why = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
        print(f"  {s/tot:6.1%} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} exc={r[ix['L1 Wavefronts Shared Excessive']]:>7} {why}")
    ex = sorted(body, key=lambda r: -int(r[ix["L1 Wavefronts Shared Excessive"]] or 0))[:8]
    print("  top excessive-wavefront instructions:")
    for r in ex:
        if int(r[ix["L1 Wavefronts Shared Excessive"]] or 0) == 0:
            break
        print(f"    {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} wf={r[ix['L1 Wavefronts Shared']]} ideal={r[ix['L1 Wavefronts Shared Ideal']]} exc={r[ix['L1 Wavefronts Shared Excessive']]}")
