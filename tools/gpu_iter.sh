#!/bin/bash
# One build->measure iteration on the GPU box: parity tests of the search,
# then the benchmark line.  Usage: tools/gpu_iter.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-"dftsp or scale or sweep"}
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/iter_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/iter_tests.log
tail -2 gpurun_out/iter_tests.log
python bench.py --steps 20 > gpurun_out/iter_bench.log 2>&1
tail -1 gpurun_out/iter_bench.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('value', round(j['value']/1e6,2), 'M ms', j['ms_per_step'], 'e2e', round(j['e2e']['value']/1e6,2), 'M', 'parity', j['parity_sample_ok'], 'clk', j['clocks'])" || tail -5 gpurun_out/iter_bench.log
