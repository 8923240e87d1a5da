"""Summarise the round-2 ncu captures (gpurun_out/prof2) into
profiles/round2_ncu.md and the per-kernel DRAM bytes bench.py reads
(profiles/ncu_summary.json)."""
import csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "gpurun_out", "prof2")
WANT = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed_op_shared_atom.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    rows = []
    for v in r[2:]:
        rows.append({a: (b, c) for a, b, c in zip(h, v, u)})
    return rows


def main():
    md = ["# Round-2 ncu captures (one B200, `scripts/profile_r2.sh`)", "",
          "`--set full --clock-control none`, one launch each (times are cold-cache, serialised",
          "and at ncu's clocks; the bench's CUDA-event times are the timing of record).", ""]
    summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    keys = {"sc_batch_screen": "sc_batch_screen", "sc_screen": "sc_screen", "sw_screen": "sw_screen",
            "trace_lane": "k_trace_lane", "decision": "k_decision"}
    for f, key in keys.items():
        rep = os.path.join(P, f + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        for i, row in enumerate(raw(rep)):
            name = row.get("Kernel Name", ("?",))[0]
            md.append(f"## {f} (launch {i}): `{name[:110]}`")
            md.append("")
            md.append("| metric | value | unit |")
            md.append("|---|---|---|")
            for w in WANT:
                if w in row:
                    md.append(f"| {w} | {row[w][0]} | {row[w][1]} |")
            md.append("")
            if i == 0:
                def val(w, scale):
                    v, unit = row[w]
                    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
                    return float(v.replace(",", "")) * mult.get(unit, 1)
                tr = val("dram__bytes_read.sum", 1) + val("dram__bytes_write.sum", 1)
                tu = row["gpu__time_duration.sum"]
                summ[key] = {"kernel": name[:120], "dram_bytes_per_launch": tr,
                             "ncu_time": [tu[0], tu[1]],
                             "source": "profiles/round2_ncu.md (scripts/profile_r2.sh)"}
    open(os.path.join(ROOT, "profiles", "round2_ncu.md"), "w").write("\n".join(md) + "\n")
    json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    print("\n".join(md[:80]))


if __name__ == "__main__":
    main()
