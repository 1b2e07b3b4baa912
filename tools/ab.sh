#!/bin/bash
# same-box A/B: tools/ab.sh NAME1 NAME2 ... (build_variants/libmotif_b200_NAME.so), 2 rounds each
cd "$(dirname "$0")/.."
for r in 1 2; do for v in "$@"; do
  echo "== $v (round $r)"
  MB_LIB_PATH=$PWD/build_variants/libmotif_b200_$v.so python tools/quick_c1.py 2>&1 | grep -E "leaf|tri_hist|rep 2" | cut -c1-60
done; done
