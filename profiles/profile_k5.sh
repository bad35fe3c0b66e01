#!/bin/bash
# ncu --set full capture of one k-5 launch: profiles/profile_k5.sh <workload> <kernel regex> <tag> [env...]
w=${1:-c2}; k=${2:-k5_pairs}; tag=${3:-r2_k5_pairs_$w}
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/$tag -f \
    python profiles/profile_target.py --workload $w --ticks 8 --warm 30 2>&1 | tail -3
python profiles/ncu_lines.py gpurun_out/$tag.ncu-rep 45 > gpurun_out/$tag.summary.txt 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>/dev/null
