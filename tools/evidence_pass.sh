#!/bin/bash
# One evidence pass on the GPU box (round 2): bench lines for configs 2/4/5
# and the reference arm, the launch list of the bench command, and one
# `ncu --set full` capture per kernel family.  Reports land in
# gpurun_out/prof/; tools/ncu_summary.py turns them into profiles/*.json here.
# Usage (from the repo root, on the box): tools/evidence_pass.sh [what...]
#   what: bench c4 c5 ref launches dftsp c5ncu wide brute k12   (default: all)
# Reports are exported to *_raw.csv / *_src.csv.gz and deleted (64 MiB pull cap).
O=gpurun_out/prof
mkdir -p $O
WHAT=${*:-"bench c4 c5 ref launches dftsp c5ncu wide brute k12"}
NCU="ncu --set full --import-source on --clock-control none"
has() { [[ " $WHAT " == *" $1 "* ]]; }
run() { local name=$1; shift; local t0=$(date +%s); timeout 900 "$@" > $O/$name.out 2> $O/$name.err; echo "$name rc=$? $(( $(date +%s) - t0 ))s"; }

has bench    && run bench python bench.py
has c5       && run bench_c5 python bench.py --config 5 --no-cpu
has c4       && run bench_c4 python bench.py --config 4 --steps 10 --warmup 3
has ref      && run ref python bench.py --impl reference
has launches && run launches ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
                    --log-file $O/launches_bench.csv python bench.py --no-cpu
has dftsp    && run ncu_dftsp $NCU -k regex:'dftsp_lock_kernel' -c 1 -o $O/dftsp -f \
                    python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e
has c5ncu    && run ncu_c5 $NCU -k regex:'dftsp_lock_kernel' -c 1 -o $O/config5 -f \
                    python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e
has wide     && run ncu_wide $NCU -k regex:'dftsp_lock_wide' -c 1 -o $O/wide -f \
                    python tools/run_workload.py --K 120 --n 20000
has brute    && run ncu_brute $NCU -k regex:'exh_(range|levels|batch)_kernel' -c 6 -o $O/brute -f \
                    python bench.py --config 4 --steps 1 --warmup 0
has k12      && run ncu_k12 $NCU -k regex:'link_kernel|admission_kernel|coeff_kernel|check_direct_kernel|check_knapsack_kernel' \
                    -c 5 -o $O/k12 -f python tools/k12_volume.py --reps 1
# gpurun copies back at most 64 MiB: keep the raw-metric and source-page
# exports (tools/ncu_summary.py, tools/ncu_lines.py read them), drop the reports
for r in $O/*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i "$r" --page raw --csv --print-units base > ${b}_raw.csv 2>/dev/null
  ncu -i "$r" --page source --csv --print-source cuda,sass 2>/dev/null | gzip -9 > ${b}_src.csv.gz
  rm -f "$r"
done
ls -la $O
