#!/bin/bash
# ncu capture of the dense k-5 gather on a large-field workload: profiles/profile_dense.sh c3
w=${1:-c3}
ncu --set full --clock-control none --import-source on -k regex:k5_writeback -s 4 -c 1 -o gpurun_out/dense_$w python profiles/profile_target.py --workload $w --ticks 2 --warm 3 2>&1 | tail -2
