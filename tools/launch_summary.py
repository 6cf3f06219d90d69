"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launches, total ms, share among the library's (hc::) kernels, average us.
Usage: python tools/launch_summary.py launches.csv [title]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, rows = rows[0], rows[1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki]
        short = name.split("(")[0].replace("void ", "")
        agg[short][0] += 1
        agg[short][1] += float(r[vi]) / 1e6  # ns -> ms
    ours = {k: v for k, v in agg.items()
            if k.startswith("hc::") or k in ("<unnamed>::k_submit", "<unnamed>::k_wait")}  # (older builds)
    tot = sum(v[1] for v in ours.values())
    print(f"# {sys.argv[2] if len(sys.argv) > 2 else path}\n")
    print("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
    for k, (n, ms) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {ms:.3f} | {100 * ms / tot:.1f} % | {1000 * ms / n:.1f} |")
    other = {k: v for k, v in agg.items() if k not in ours}
    if other:
        print("\nnot ours (input generation / torch fills outside the timed region): " +
              ", ".join(f"`{k}` x{v[0]}" for k, v in other.items()))


if __name__ == "__main__":
    main()
