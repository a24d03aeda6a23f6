#!/bin/bash
# Build the engine from a git revision (or the working tree, rev "WT") with extra nvcc
# defines into variants/<name>/libstda_b200.so, for A/B timing via STDA_LIB_PATH.
# usage: tools/build_variant.sh <name> <rev|WT> [-DMACRO ...]
set -e
name=$1; rev=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
if [ "$rev" = "WT" ]; then
  cp -r "$root/paper_2307_09063_b200/csrc" "$tmp/csrc"; mkdir -p "$tmp/include"; cp "$root/include/"*.h "$tmp/include/"
else
  (cd "$root" && git archive "$rev" paper_2307_09063_b200/csrc include) | tar -x -C "$tmp"
  mv "$tmp/paper_2307_09063_b200/csrc" "$tmp/csrc"
fi
mkdir -p "$tmp/pkg"; mv "$tmp/csrc" "$tmp/pkg/csrc"; rm -rf "$tmp/pkg/csrc/build" "$tmp/pkg/csrc/../libstda_b200.so"
mkdir -p "$tmp/include"
make -s -C "$tmp/pkg/csrc" -j 8 FLAGS="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $*" \
  HDRS="$(cd "$tmp/pkg/csrc" && ls *.cuh | tr '\n' ' ')" > /dev/null
mkdir -p "$root/variants/$name"
cp "$tmp/pkg/libstda_b200.so" "$root/variants/$name/"
rm -rf "$tmp"
echo "variants/$name/libstda_b200.so"
