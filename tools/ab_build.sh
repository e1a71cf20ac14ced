#!/bin/bash
# Build libhsk.so of a git revision into _exp/ab/libhsk_<tag>.so for same-box
# A/B timing:  HSK_LIB=_exp/ab/libhsk_<tag>.so python tools/kbench.py ...
set -e
rev=${1:?revision}; tag=${2:-$rev}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2302_01977_b200 include | tar -x -C "$tmp"
(cd "$tmp" && python -c "import paper_2302_01977_b200.build as b; b.build()" > /dev/null)
mkdir -p "$root/_exp/ab"
cp "$tmp/paper_2302_01977_b200/libhsk.so" "$root/_exp/ab/libhsk_$tag.so"
rm -rf "$tmp"
echo "$root/_exp/ab/libhsk_$tag.so"
