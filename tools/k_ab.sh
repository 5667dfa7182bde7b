#!/bin/bash
# kernel rate of tools/run_workload.py across library variants: tools/k_ab.sh "ARGS" v1 v2 ...
args=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v.so; fi
  echo "$v $args: $(EB_LIB_PATH=$lib timeout 300 python tools/run_workload.py $args 2>&1 | tail -1)"
done
