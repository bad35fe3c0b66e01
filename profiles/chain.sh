#!/bin/bash
# chained launches (programmatic dependent launch, sfc_internal.cuh) on / off: tick time per workload
for spec in "c1:SFC_CHAIN=1" "c1:SFC_CHAIN=0" "c2:SFC_CHAIN=1" "c2:SFC_CHAIN=0" "paper1000:SFC_CHAIN=1" "paper1000:SFC_CHAIN=0" "c4r:SFC_CHAIN=1" "c4r:SFC_CHAIN=0"; do
  w=${spec%%:*}; envs=${spec#*:}
  env $envs python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ch_$w.json 2> gpurun_out/ch_$w.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/ch_$w.json"))
    print("$w [$envs] tick_us %.2f" % d["tick_us"], "value %.3e" % d["value"], "e2e %.3e" % d["e2e"]["value"], "launches", d.get("gpu_launches"))
except Exception as e:
    print("$w [$envs] failed", e); print(open("gpurun_out/ch_$w.err").read()[-1500:])
PY
done
