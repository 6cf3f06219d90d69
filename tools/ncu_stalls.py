"""Stall-reason breakdown of one kernel in an .ncu-rep, by SASS region.

usage: python tools/ncu_stalls.py REP [block]   (block = #SASS instructions per region)"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 400
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
S = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
ex = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[S]) for r in data)
print(f"total samples {tot}")
for k in range(0, len(data), blk):
    b = data[k:k + blk]
    s = sum(int(r[S]) for r in b)
    if s < tot * 0.02:
        continue
    rs = {h: sum(int(r[hdr.index(h)] or 0) for r in b) for h in reasons}
    top = sorted(rs.items(), key=lambda x: -x[1])[:4]
    ops = {}
    for r in b:
        m = re.match(r'\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+)', r[src])
        if m and int(r[ex] or 0) > 0:
            op = m.group(1)
            if op in ("ATOMS", "STG", "LDG", "LDS", "STS", "SHFL", "BAR", "LDGSTS", "RED", "ATOM"):
                ops[op] = ops.get(op, 0) + 1
    print(f"[{k:6d}] {100*s/tot:5.1f}%  inst={sum(int(r[ex] or 0) for r in b):>10d}  "
          + " ".join(f"{h[6:]}={100*v/max(s,1):.0f}%" for h, v in top) + f"  {ops}")
