"""Summarise ncu reports (--set full) into a markdown table: duration, DRAM
bytes, throughput fractions, tensor-pipe / shared-pipe activity per kernel.

    python scripts/ncu_summarize.py out.md rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    res = []
    for v in r[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        res.append((d.get("Kernel Name", "?"), {k: (d.get(k, ""), u.get(k, "")) for k, _ in METRICS}))
    return res


def main():
    out = sys.argv[1]
    lines = ["| report | kernel | " + " | ".join(n for _, n in METRICS) + " |",
             "|---" * (len(METRICS) + 2) + "|"]
    for rep in sys.argv[2:]:
        for name, d in rows(rep):
            short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
            short = short.replace("moe::", "").replace("unnamed>::", "")
            cells = [f"{d[k][0]} {d[k][1]}".strip() for k, _ in METRICS]
            lines.append(f"| {rep.split('/')[-1]} | {short[:40]} | " + " | ".join(cells) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
