#!/usr/bin/env python3
"""Per-phase / per-line instruction and stall-sample breakdown of an ncu
report's source page (cuda,sass).  Usage: tools/ncu_lines.py SRC.csv UNITS [top]"""
import csv
import re
import sys


def load(path):
    rows, f, hdr = [], None, None
    if path.endswith(".gz"):
        import gzip
        fh = gzip.open(path, "rt")
    else:
        fh = open(path)
    for r in csv.reader(fh):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
            ie = int(d["Instructions Executed"])
            th = int(d["Thread Instructions Executed"])
        except (KeyError, ValueError):
            continue
        rows.append((f, int(r[0]), s, ie, th, r[1].strip()[:100]))
    return rows


def phases(src="paper_2405_07140_b200/csrc/eb_dftsp.cu"):
    marks = [("level_counts", r"^// Full-traversal node counts"), ("misc", r"^// Phase barrier of the lockstep"),
             ("U tables", r"---- U:"), ("S search", r"---- S:"), ("C counts", r"---- C:"),
             ("write_status", r"^__device__ __noinline__ void write_status"),
             ("setup", r"setup: per request"), ("per-d tables", r"per pool width d: class"),
             ("search dispatch", r"---------------- search"), ("finish", r"---------------- finish"),
             ("kernels", r"^template <bool PRUNE, bool INCL, bool EXACT, int ALGO, int NI>\s*$")]
    lines = open(src).read().split("\n")
    starts = []
    for name, pat in marks:
        idx = [i + 1 for i, l in enumerate(lines) if re.search(pat, l)]
        starts.append((idx[-1] if name == "kernels" else idx[0], name))
    starts.sort()
    return [(0, "helpers")] + starts


def main():
    rows = load(sys.argv[1])
    units = float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    ts = sum(x[2] for x in rows)
    ti = sum(x[3] for x in rows)
    print(f"warp-inst/unit {ti / units:.1f}  threads/inst {sum(x[4] for x in rows) / max(ti, 1):.2f}")
    ph = phases()
    agg = {}
    for f, ln, s, ie, th, _ in rows:
        name = f
        if f == "eb_dftsp.cu":
            name = [n for st, n in ph if st <= ln][-1]
        a = agg.setdefault(name, [0, 0, 0])
        a[0] += s
        a[1] += ie
        a[2] += th
    for k, (s, ie, th) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} samples {100 * s / ts:5.1f}%  inst/unit {ie / units:8.1f}  lanes {th / max(ie, 1):5.1f}")
    print("--- top lines by instructions")
    for x in sorted(rows, key=lambda x: -x[3])[:top]:
        print(f"{x[0][:14]:14s}{x[1]:5d} i/unit={x[3] / units:7.1f} s={100 * x[2] / ts:5.2f}% lanes={x[4] / max(x[3], 1):4.1f} {x[5]}")


if __name__ == "__main__":
    main()
