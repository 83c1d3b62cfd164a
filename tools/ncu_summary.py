"""Summarise one kernel of an .ncu-rep (ncu --set full) as JSON for profiles/.

  python tools/ncu_summary.py gpurun_out/ncu_i8w_r02.ncu-rep "config text" > profiles/ncu_....json
"""
import csv
import json
import subprocess
import sys

rep, config = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}


def val(name, scale=1.0):
    i = col.get(name)
    if i is None or vals[i] == "":
        return None
    v = float(vals[i].replace(",", ""))
    u = units[i]
    mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-3, "ms": 1.0, "s": 1e3, "ns": 1e-6}.get(u, 1.0)
    return v * mult * scale


out = {
    "round": 2,
    "kernel": vals[col["Kernel Name"]],
    "config": config,
    "gpu_time_ms": val("gpu__time_duration.sum"),
    "dram_read_bytes_per_launch": val("dram__bytes_read.sum"),
    "dram_write_bytes_per_launch": val("dram__bytes_write.sum"),
    "fp64_pipe_active_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "imma_inst_pct": val("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active"),
    "dmma_inst_pct": val("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": val("launch__registers_per_thread"),
    "warp_instructions": val("smsp__inst_executed.sum"),
    "stalls_per_issue": {h.split("issue_stalled_")[1].split("_per_issue")[0]: float(vals[i])
                         for h, i in col.items()
                         if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                         and vals[i] not in ("", "0") and float(vals[i]) >= 0.05},
    "source": f"{rep} (ncu --set full --clock-control none --import-source on)",
}
print(json.dumps(out, indent=1))
