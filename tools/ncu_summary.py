#!/usr/bin/env python3
"""Summarise an ncu --set full report (one kernel launch) into the JSON kept
under profiles/: duration, DRAM bytes, warp instructions, issue activity,
occupancy, registers, stall breakdown.  Usage:
  tools/ncu_summary.py REPORT.ncu-rep|RAW.csv KERNEL_REGEX UNITS_PER_LAUNCH [--launch i]"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "sm_clock_ghz": ("smsp__cycles_elapsed.avg.per_second", 1e-9),
    "dram_bytes_read": ("dram__bytes_read.sum", 1.0),
    "dram_bytes_write": ("dram__bytes_write.sum", 1.0),
    "warp_instructions": ("smsp__inst_executed.sum", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "ipc_per_sm": ("sm__inst_executed.avg.per_cycle_active", 1.0),
    "threads_per_warp_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "block": ("launch__block_size", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "smem_per_block_kb": ("launch__shared_mem_per_block_dynamic", 1.0 / 1024),
    "occupancy_warps_pct": ("sm__maximum_warps_per_active_cycle_pct", 1.0),
}
STALLS = ["barrier", "branch_resolving", "dispatch_stall", "long_scoreboard", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "no_instruction", "not_selected", "selected", "short_scoreboard", "wait", "sleeping"]


def main():
    rep, kern, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
    launch = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
    if rep.endswith(".csv"):      # a `--page raw --csv --print-units base` export (tools/evidence_pass.sh)
        import re
        rows = list(csv.reader(open(rep)))
        hdr = rows[0]
        kn = hdr.index("Kernel Name")
        data = [r for r in rows[2:] if re.search(kern, r[kn])]
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "-k",
                              f"regex:{kern}"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, data = rows[0], rows[2:]
    row = dict(zip(hdr, data[launch]))

    def val(name):
        v = row.get(name, "")
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return None
    s = {"kernel": row.get("Kernel Name"), "units_per_launch": units}
    for k, (m, scale) in METRICS.items():
        v = val(m)
        s[k] = None if v is None else round(v * scale, 6)
    if s["dram_bytes_read"] is not None:
        s["dram_bytes_per_launch"] = s["dram_bytes_read"] + s["dram_bytes_write"]
    if s["warp_instructions"]:
        s["warp_instructions_per_unit"] = round(s["warp_instructions"] / units, 3)
    st = {}
    for n in STALLS:
        v = val(f"smsp__average_warps_issue_stalled_{n}_per_issue_active.ratio")
        if v is not None:
            st[n] = round(v, 3)
    s["stalls_per_issue"] = st
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
