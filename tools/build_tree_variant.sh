#!/bin/bash
# A/B build of the library with some sources taken from a git revision:
#   tools/build_tree_variant.sh <name> <rev> <csrc file> [<csrc file> ...]
# -> paper_1909_04153_b200/lib/variants/<name>.so (load with BSQ_LIB=...)
set -e
name=$1; rev=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r "$root/paper_1909_04153_b200" "$root/include" "$tmp/"
rm -rf "$tmp/paper_1909_04153_b200/lib"
for f in "$@"; do
  git -C "$root" show "$rev:paper_1909_04153_b200/csrc/$f" > "$tmp/paper_1909_04153_b200/csrc/$f"
done
(cd "$tmp" && python -m paper_1909_04153_b200.build --force > /dev/null 2>&1)
mkdir -p "$root/paper_1909_04153_b200/lib/variants"
cp "$tmp/paper_1909_04153_b200/lib/libbsq.so" "$root/paper_1909_04153_b200/lib/variants/$name.so"
rm -rf "$tmp"
echo "$root/paper_1909_04153_b200/lib/variants/$name.so"
