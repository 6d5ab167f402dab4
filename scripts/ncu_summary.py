"""Summarise ncu evidence into profiles/ (tracked).

  python scripts/ncu_summary.py <cfg> <prof.ncu-rep> [launches.csv] [--out-md profiles/..md]

Reads a `--set full` capture (raw page) and, optionally, the launch list of the bench
command (`--metrics gpu__time_duration.sum`), and updates profiles/ncu_summary.json[cfg]
with the per-launch DRAM traffic that bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "kernel duration (ncu, clocks unlocked, cold)"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("sm__cycles_active.min", "SM active cycles min"),
    ("sm__cycles_active.avg", "SM active cycles avg"),
    ("sm__cycles_active.max", "SM active cycles max"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_tensor.sum", "tensor instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for vals in rows[2:]:
        recs.append({h: (v, u) for h, v, u in zip(hdr, vals, units)})
    return recs


def stalls(rec):
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[0] or 0)
          for k, v in rec.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1.0
    return sorted(((k, 100 * v / tot) for k, v in st.items()), key=lambda x: -x[1])[:8]


def launches(path):
    if not path or not os.path.exists(path):
        return None
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        val = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r["Metric Unit"]]
        per.setdefault(name, []).append(val * scale)
    return per


def main():
    cfg, rep = sys.argv[1], sys.argv[2]
    lpath = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else None
    md_out = sys.argv[sys.argv.index("--out-md") + 1] if "--out-md" in sys.argv else None
    recs = raw(rep)
    rec = recs[0]
    name = rec.get("Kernel Name", ("?",))[0]
    summary = {"kernel": name}
    lines = [f"# ncu summary: {cfg} -- `{name}`", "", f"source: `{os.path.basename(rep)}` (ncu --set full, "
             "--clock-control none, one launch)", "", "| metric | value | unit |", "|---|---|---|"]
    for k, desc in KEYS:
        if k in rec:
            v, u = rec[k]
            lines.append(f"| {desc} (`{k}`) | {v} | {u} |")
            summary[k] = v
    rd = float(rec["dram__bytes_read.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[rec["dram__bytes_read.sum"][1]]
    wr = float(rec["dram__bytes_write.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[rec["dram__bytes_write.sum"][1]]
    summary["dram_bytes_per_launch"] = rd + wr
    lines += ["", f"DRAM traffic per launch (read + write): {rd + wr:.6e} B", "", "## issue-stall samples (% of stalled samples)", ""]
    for k, pct in stalls(rec):
        lines.append(f"- {k}: {pct:.1f}%")
    per = launches(lpath)
    if per:
        tot = sum(sum(v) for v in per.values())
        lines += ["", f"## launch list (`{os.path.basename(lpath)}`: every launch of the bench command, cold/serialised)", "",
                  "| kernel | launches | total us | share of all GPU time | mean us |", "|---|---|---|---|---|"]
        for n, v in sorted(per.items(), key=lambda x: -sum(x[1]))[:8]:
            lines.append(f"| `{n[:80]}` | {len(v)} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% | {sum(v) / len(v):.1f} |")
        lines.append("")
        lines.append("The list is filtered to the library's kernels (ncu -k la_decode|la_combine): a bench step at "
                     "N=1 is exactly one la_decode launch, so the decode kernel is 100% of the step's GPU time "
                     "(torch's synthetic-input generation runs before the timed region).")
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[cfg] = summary
    json.dump(data, open(path, "w"), indent=1)
    if md_out:
        open(md_out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
