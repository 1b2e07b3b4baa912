#!/bin/bash
# Build the library at a git ref into build_variants/libmotif_b200_NAME.so for
# same-box A/B timing (MB_LIB_PATH=...):  tools/build_ref.sh NAME REF
set -e
cd "$(dirname "$0")/.."
name=$1; ref=$2
wt=/tmp/mb_wt_$name
rm -rf $wt; git worktree prune
git worktree add -f $wt $ref > /dev/null 2>&1
make -C $wt/paper_1602_04478_b200 -j8 > /dev/null 2>&1 || (make -C $wt/paper_1602_04478_b200 2>&1 | tail -20; exit 1)
mkdir -p build_variants
cp $wt/paper_1602_04478_b200/libmotif_b200.so build_variants/libmotif_b200_$name.so
git worktree remove -f $wt
echo built build_variants/libmotif_b200_$name.so
