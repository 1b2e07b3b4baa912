#!/bin/bash
# same-box A/B of environment switches: tools/ab_env.sh "" "MB_X=1" ... (2 rounds each)
cd "$(dirname "$0")/.."
for r in 1 2; do for v in "$@"; do
  echo "== [$v] (round $r)"
  env $v python tools/quick_c1.py 2>&1 | grep -E "leaf|tri_hist|rep 2" | cut -c1-60
done; done
