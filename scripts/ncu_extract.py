"""Summarise ncu --set full reports (one launch each): the metrics the
profiles/ tables quote, as a markdown table and a JSON extract.
usage: ncu_extract.py OUT_PREFIX name=report.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "kernel": "Kernel Name",
    "gpu_time_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "warp_inst": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_per_sched": "smsp__warps_active.avg.per_cycle_active",
    "warps_eligible_per_sched": "smsp__warps_eligible.avg.per_cycle_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_pct_peak": "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
}
UNITS = {"gpu__time_duration.sum": 1e-6, "dram__bytes_read.sum": 1.0, "dram__bytes_write.sum": 1.0}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    v = rows[2] if len(rows) > 2 else rows[1]
    return dict(zip(h, v))


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


out, reps = sys.argv[1], sys.argv[2:]
res = {}
for r in reps:
    name, path = r.split("=", 1)
    d = raw(path)
    e = {}
    for k, m in KEYS.items():
        val = num(d.get(m, "nan"))
        if m == "gpu__time_duration.sum" and isinstance(val, float):
            val = val * 1e-6  # ns -> ms
        e[k] = val
    res[name] = e
json.dump(res, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as f:
    f.write("| config | kernel | gpu time ms | DRAM read+write | warp instr | issue busy % | warps active / eligible per scheduler | regs | L2 hit % | DRAM % peak |\n|---|---|---|---|---|---|---|---|---|---|\n")
    for name, e in res.items():
        rw = (e["dram_read_bytes"] + e["dram_write_bytes"]) if isinstance(e["dram_read_bytes"], float) else "?"
        k = str(e["kernel"]).split("(")[0]
        f.write(f"| {name} | `{k}` | {e['gpu_time_ms']:.3f} | {rw/1e6:.1f} MB | {e['warp_inst']/1e6:.1f} M | "
                f"{e['issue_active_pct']:.1f} | {e['warps_active_per_sched']:.2f} / {e['warps_eligible_per_sched']:.2f} | "
                f"{int(e['regs'])} | {e['l2_hit_pct']:.1f} | {e['dram_pct_peak']:.1f} |\n")
print(open(out + ".md").read())
