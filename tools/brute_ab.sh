#!/bin/bash
# A/B the config-4 bench line (brute force K=32) across library variants.
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v.so; fi
  EB_LIB_PATH=$lib timeout 600 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/c4_$v.json 2> gpurun_out/c4_$v.err
  python -c "import json; j=json.loads(open('gpurun_out/c4_$v.json').read().strip().splitlines()[-1]); print('$v', j['value'], 'inst/s', j['ms_per_step'], 'ms/step checked/s %.3g' % j['checked_subsets_per_s'], j['results'][:2])" || tail -3 gpurun_out/c4_$v.err
done
