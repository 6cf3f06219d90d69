"""Hottest SASS instructions of one kernel in an .ncu-rep (warp-stall samples).
usage: python tools/ncu_hot.py REP KERNEL_REGEX [top]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
blocks, cur = [], []
for l in lines:
    if l.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [l]
    else:
        cur.append(l)
if cur:
    blocks.append(cur)
b = blocks[0]
rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
hdr, data = rows[0], rows[1:]
S, E = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(int(r[S] or 0) for r in data)
print(f"{b[0][:90]}  total samples {tot}")
idx = sorted(range(len(data)), key=lambda i: -int(data[i][S] or 0))[:top]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {int(r[S]):6d} {100*int(r[S])/tot:5.1f}%  {r[1].strip()[:70]}")
