#!/bin/bash
# config-4 bench line under EB_BRUTE_CHUNKS / EB_BRUTE_MINCHUNK settings: "C:M" pairs
for cm in "$@"; do
  c=${cm%:*}; m=${cm#*:}
  EB_BRUTE_CHUNKS=$c EB_BRUTE_MINCHUNK=$m timeout 600 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/c4e.json 2> gpurun_out/c4e.err
  python -c "import json; j=json.loads(open('gpurun_out/c4e.json').read().strip().splitlines()[-1]); print('$cm', j['value'], 'inst/s', j['ms_per_step'], 'ms/step checked/s %.3g' % j['checked_subsets_per_s'])" || tail -3 gpurun_out/c4e.err
done
