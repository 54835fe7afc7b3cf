#!/bin/bash
# Build libmaxmin.so of a git ref in a temporary worktree and copy it into the
# package as lib_<name>.so (A/B timing against the working tree's build).
#   tools/build_ref_lib.sh <ref> <name>
set -e
ref=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/maxmin_wt_$name
rm -rf "$wt"; git -C "$root" worktree prune
git -C "$root" worktree add -f "$wt" "$ref" > /dev/null
(cd "$wt" && python -c "from paper_cs_0610046_b200 import _build; _build.build(force=True)" > /dev/null 2>&1)
cp "$wt/paper_cs_0610046_b200/libmaxmin.so" "$root/paper_cs_0610046_b200/lib_$name.so"
git -C "$root" worktree remove --force "$wt"
echo "$root/paper_cs_0610046_b200/lib_$name.so"
