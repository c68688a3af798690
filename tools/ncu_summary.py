"""Summarise ncu artefacts for profiles/:
  python tools/ncu_summary.py full  <report.ncu-rep> <out.md> [config]   -- one --set full capture
  python tools/ncu_summary.py launches <launches.csv> <out.csv>          -- launch list (gpu__time_duration)
The `full` mode also updates profiles/core_traffic.json (dram bytes per launch of the core
kernel for `config`), which bench.py reports as roofline.traffic."""
import csv, io, json, os, subprocess, sys, collections

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle / issue"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch_resolving / issue"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall no_instruction / issue"),
]

def to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return float(v) * f if f else None

def full(rep, out, config="llama3"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full: `{os.path.basename(rep)}`", ""]
    for row in rows[2:]:
        name = row[h.index("Kernel Name")]
        lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        for k, label in KEYS:
            if k in d:
                lines.append(f"| {label} (`{k}`) | {d[k]} | {u[k]} |")
        rd = to_bytes(d.get("dram__bytes_read.sum", 0), u.get("dram__bytes_read.sum"))
        wr = to_bytes(d.get("dram__bytes_write.sum", 0), u.get("dram__bytes_write.sum"))
        if "core_kernel" in name and rd is not None and wr is not None:
            tj = os.path.join(os.path.dirname(out), "core_traffic.json")
            prof = json.load(open(tj)) if os.path.exists(tj) else {}
            prof[config] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                            "source": os.path.basename(rep)}
            json.dump(prof, open(tj, "w"), indent=1)
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")

def launches(src, out):
    rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
    h = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        n = r[h.index("Kernel Name")]
        v = float(r[h.index("Metric Value")].replace(",", ""))
        agg.setdefault(n, []).append(v)
    ours = lambda n: "msd::" in n or any(k in n for k in ("core_kernel", "tail_kernel", "rollback_kernel", "exp_table_kernel", "pool_kernel", "draft_kernel"))
    tot = sum(sum(v) for n, v in agg.items() if ours(n))
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "avg_ns", "min_ns", "max_ns", "share_of_msd_time"])
        for n, v in agg.items():
            if ours(n):
                w.writerow([n, len(v), round(sum(v) / len(v)), round(min(v)), round(max(v)), round(sum(v) / tot, 4)])
        others = [x for n, v in agg.items() if not ours(n) for x in v]
        w.writerow(["(torch input generation, outside the timed region)", len(others), "", "", "", ""])

if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "llama3")
    else:
        launches(sys.argv[2], sys.argv[3])
