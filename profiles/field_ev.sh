#!/bin/bash
# field kernel: events looked up per loop trip (SFC_FIELD_EV), rebuilt on the box for each value
f=paper_1803_04782_b200/csrc/sfc_k5_field.cu
for ev in "(LAZY ? 1 : 4)" "(LAZY ? 2 : 4)"; do
  sed -i "s/^#define SFC_FIELD_EV .*/#define SFC_FIELD_EV $ev/" $f
  python -c "from paper_1803_04782_b200 import build; build.build_cuda(verbose=False)" || exit 1
  echo "== EV $ev"
  bash profiles/field_try.sh ev c3 c3:SFC_K5_FIELD_WARPS=16 c3:SFC_K5_FIELD_WARPS=4 "c3:SFC_K5_FIELD_NK=3 SFC_K5_FIELD_WARPS=4" "c3:SFC_K5_FIELD_NK=3 SFC_K5_FIELD_WARPS=8" c3:SFC_K5_FIELD_LAZY=0
done
