#!/bin/bash
# field-kernel tuning: tick / k-5 times of the large-field workloads under a few shapes
tag=${1:-ft}; shift
for spec in "$@"; do
  w=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
  env $envs python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/${tag}_$w.json 2> gpurun_out/${tag}_$w.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/${tag}_$w.json"))
    print("$w [$envs]", "tick_us %.1f" % d["tick_us"], "k5 %.1f" % d["phase_us_per_tick"]["k5"], "path", d["config"]["k5_path"], "frac %.3f" % d["roofline"]["frac"])
except Exception as e:
    print("$w [$envs] failed", e); print(open("gpurun_out/${tag}_$w.err").read()[-1500:])
PY
done
