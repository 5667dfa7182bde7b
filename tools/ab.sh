#!/bin/bash
# A/B the kernel-only bench value across library variants (tools/variants.sh):
#   tools/ab.sh [bench args] -- default r96w20 ...
args=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do args+=("$1"); shift; done
shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v.so; fi
  EB_LIB_PATH=$lib timeout 600 python bench.py --no-cpu --no-e2e "${args[@]}" > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json,sys; j=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(j['value']/1e6,2), 'M inst/s', j['ms_per_step'], 'ms parity', j['parity']['ok'], 'issue', j['roofline']['issue'].get('peak_measured'))" || tail -3 gpurun_out/ab_$v.err
done
