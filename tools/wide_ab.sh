for v in prev default w2; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v.so; fi
  for K in 80 120 200; do echo "$v K=$K $(EB_LIB_PATH=$lib timeout 300 python tools/run_workload.py --K $K --n 20000 2>&1 | tail -1)"; done
done
