"""Summarise an .ncu-rep (ncu -i ... --page raw --csv) into a compact markdown table."""
import csv, io, subprocess, sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu summary of `{rep.split('/')[-1]}`", "",
             "| kernel | " + " | ".join(n for _, n in WANT) + " |",
             "|---|" + "---|" * len(WANT)]
    for d in data:
        name = d[hdr.index("Kernel Name")][:48]
        vals = []
        for m, _ in WANT:
            if m in hdr:
                i = hdr.index(m)
                vals.append(f"{d[i]} {units[i]}".strip())
            else:
                vals.append("-")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
