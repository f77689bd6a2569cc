"""Summarise ncu reports (development aid): per kernel launch, the metrics
the roofline / DESIGN.md cite.  Usage: python tools/ncu_summary.py a.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
}
UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}

out = []
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"report": rep.split("/")[-1], "kernel": r[hdr.index("Kernel Name")][:120]}
        for i, name in enumerate(hdr):
            if name in WANT:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if WANT[name] == "duration":
                    v *= UNITS.get(u, 1.0) * 1e3
                    d["duration_ms"] = v
                elif WANT[name].startswith("dram_r") or WANT[name].startswith("dram_w"):
                    d[WANT[name] + "_bytes"] = v * UNITS.get(u, 1.0)
                else:
                    d[WANT[name]] = v
        stalls = {}
        for i, name in enumerate(hdr):
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in name:
                try:
                    stalls[name.split("stalled_")[1]] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        if "duration_ms" in d and "dram_read_bytes" in d:
            d["dram_gbs"] = (d["dram_read_bytes"] + d.get("dram_write_bytes", 0)) / (d["duration_ms"] * 1e-3) / 1e9
        out.append(d)
print(json.dumps(out, indent=1))
