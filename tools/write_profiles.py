#!/usr/bin/env python3
"""Turn an evidence pass (tools/evidence_pass.sh -> gpurun_out/prof/) into the
committed profiles/ summaries: ncu_{dftsp,config5,wide}_summary.json (one
launch each), ncu_{brute,k12}_summary.json (every captured launch),
r02_{dftsp,config5}_phases.txt, r02_bench_lines.jsonl and the launch list.
Usage: tools/write_profiles.py [PROF_DIR] [what ...]   what: dftsp c5 wide brute k12 bench launches"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
P = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof")
WHAT = set(sys.argv[2:]) or {"dftsp", "c5", "wide", "brute", "k12", "bench", "launches"}
OUT = os.path.join(ROOT, "profiles")
NCU = "ncu --set full --import-source on --clock-control none"


def summ(raw, kern, units):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), os.path.join(P, raw), kern,
                          str(units)], capture_output=True, text=True, check=True).stdout
    return json.loads(out)


def one(raw, kern, units, name, cmd, notes):
    from paper_2405_07140_b200._build import source_hash
    j = summ(raw, kern, units)
    out = {"round": 2, "kernel": j.pop("kernel"), "command": cmd, "source_hash": source_hash(),
           "instances_per_launch": j.pop("units_per_launch")}
    out.update(j)
    out["warp_instructions_per_instance"] = out.pop("warp_instructions_per_unit")
    out["notes"] = notes
    with open(os.path.join(OUT, name), "w") as fh:
        json.dump(out, fh, indent=1)
    print(name, out["duration_ms"], "ms", out["warp_instructions_per_instance"], "warp-inst/unit",
          out["issue_active_pct"], "% issue")


M = {"duration_ms": ("gpu__time_duration.sum", 1e-6), "dram_bytes_read": ("dram__bytes_read.sum", 1),
     "dram_bytes_write": ("dram__bytes_write.sum", 1), "warp_instructions": ("smsp__inst_executed.sum", 1),
     "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
     "threads_per_warp_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
     "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
     "registers": ("launch__registers_per_thread", 1), "grid": ("launch__grid_size", 1),
     "block": ("launch__block_size", 1), "dram_gb_s": ("dram__bytes.sum.per_second", 1e-9),
     "local_load_sectors": ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", 1)}
STALLS = ["barrier", "branch_resolving", "long_scoreboard", "math_pipe_throttle", "no_instruction", "not_selected",
          "selected", "short_scoreboard", "wait", "lg_throttle", "mio_throttle"]


def launches(raw):
    r = list(csv.reader(open(os.path.join(P, raw))))
    h = r[0]
    out = []
    for x in r[2:]:
        d = dict(zip(h, x))
        s = {"kernel": d["Kernel Name"]}
        for k, (m, sc) in M.items():
            try:
                s[k] = round(float(d[m].replace(",", "")) * sc, 4)
            except (KeyError, ValueError):
                s[k] = None
        s["stalls_per_issue"] = {n: round(float(d[f"smsp__average_warps_issue_stalled_{n}_per_issue_active.ratio"]), 3)
                                 for n in STALLS
                                 if d.get(f"smsp__average_warps_issue_stalled_{n}_per_issue_active.ratio", "")}
        out.append(s)
    return out


def main():
    if "dftsp" in WHAT:
        one("dftsp_raw.csv", "dftsp_lock_kernel", 1e6, "ncu_dftsp_summary.json",
            f"{NCU} -k regex:dftsp_lock_kernel -c 1 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e",
            "round 2 capture (tools/evidence_pass.sh), first dftsp_lock_kernel launch, 10^6 config-2 instances; "
            "per-line breakdown: profiles/r02_dftsp_phases.txt")
        with open(os.path.join(OUT, "r02_dftsp_phases.txt"), "w") as fh:
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"),
                            os.path.join(P, "dftsp_src.csv.gz"), "1000000", "40"], stdout=fh, check=True)
    if "c5" in WHAT:
        one("config5_raw.csv", "dftsp_lock_kernel", 1e6, "ncu_config5_summary.json",
            f"{NCU} -k regex:dftsp_lock_kernel -c 1 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e",
            "round 2 capture, config 5 (tight-memory OPT-13B w4a16, 5 output classes), 10^6 instances; "
            "per-line: profiles/r02_config5_phases.txt")
        with open(os.path.join(OUT, "r02_config5_phases.txt"), "w") as fh:
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"),
                            os.path.join(P, "config5_src.csv.gz"), "1000000", "40"], stdout=fh, check=True)
    if "wide" in WHAT:
        one("wide_raw.csv", "dftsp_lock_wide", 2e4, "ncu_wide_summary.json",
            f"{NCU} -k regex:dftsp_lock_wide -c 1 python tools/run_workload.py --K 120 --n 20000",
            "round 2 capture, leaf-parallel wide pass (NI=4 kernel for <= 128 candidates), 2*10^4 instances K=120")
    if "brute" in WHAT:
        with open(os.path.join(OUT, "ncu_brute_summary.json"), "w") as fh:
            json.dump({"capture": f"round 2, {NCU} -k regex:'exh_(range|levels|batch)_kernel' -c 6 python bench.py "
                                  "--config 4 --steps 1 --warmup 0 (K=32 adversarial family, synth.brute_family; the "
                                  "live-level kernel, then one exh_range_kernel launch per live level)",
                       "launches": launches("brute_raw.csv")}, fh, indent=1)
    if "k12" in WHAT:
        with open(os.path.join(OUT, "ncu_k12_summary.json"), "w") as fh:
            json.dump({"capture": f"round 2, {NCU} -c 5 python tools/k12_volume.py --reps 1 (config-2 workload: "
                                  "10^6 instances x 20 rows = 2e7 rows, EB_MEM_DEVICE)",
                       "launches": launches("k12_raw.csv")}, fh, indent=1)
    if "bench" in WHAT:
        lines = []
        for f in ("bench", "bench_c4", "bench_c5", "ref"):
            p = os.path.join(P, f + ".out")
            if os.path.exists(p):
                ls = [x for x in open(p).read().splitlines() if x.startswith("{")]
                if ls:
                    lines.append(ls[-1])
        with open(os.path.join(OUT, "r02_bench_lines.jsonl"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
    if "launches" in WHAT and os.path.exists(os.path.join(P, "launches_bench.csv")):
        import shutil
        shutil.copy(os.path.join(P, "launches_bench.csv"), os.path.join(OUT, "r02_launches_bench.csv"))


if __name__ == "__main__":
    main()
