#!/bin/bash
# Build the library of a git revision (default HEAD) as variant libecho_b200_<name>.so for A/B runs.
#   tools/build_ref_variant.sh [rev] [name]
set -e
REV=${1:-HEAD}; NAME=${2:-head}
WT=/tmp/echo_wt_$NAME
rm -rf $WT; git worktree prune
git worktree add -f --detach $WT $REV > /dev/null 2>&1
(cd $WT && python -m paper_1810_04597_b200.build > /dev/null)
cp $WT/paper_1810_04597_b200/libecho_b200.so paper_1810_04597_b200/libecho_b200_$NAME.so
git worktree remove --force $WT
echo "built paper_1810_04597_b200/libecho_b200_$NAME.so from $REV"
