#!/bin/bash
# quick check on the GPU box: k-5 parity subset, then tick / phase times of the small-field workloads
tag=${1:-q}; shift
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pairs or extra or golden or acceptance3" 2>&1 | tail -3
for w in ${@:-c2 paper1000 c1 c4r}; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/${tag}_bench_$w.json"))
    print("$w", "tick_us %.1f" % d["tick_us"], {k: round(v,1) for k,v in d["phase_us_per_tick"].items()}, "value %.3g e2e %.3g frac %.3f path %s" % (d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["config"]["k5_path"]))
except Exception as e:
    print("$w failed", e); print(open("gpurun_out/${tag}_bench_$w.err").read()[-2000:])
PY
done
