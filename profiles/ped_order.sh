#!/bin/bash
# per-pedestrian kernels in position order (PedArrays::order) against id order: phase times per workload
for w in paper1000 c2 c4 c5 c3; do
  for o in 1 0; do
    SFC_PED_ORDER=$o python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/po_${w}_$o.json 2> gpurun_out/po_${w}_$o.err
    python - <<PY
import json
try:
    d=json.load(open("gpurun_out/po_${w}_$o.json"))
    print("$w order=$o tick_us %.1f" % d["tick_us"], d["phase_us_per_tick"], "value %.3e" % d["value"])
except Exception as e:
    print("$w order=$o failed", e); print(open("gpurun_out/po_${w}_$o.err").read()[-1500:])
PY
  done
done
