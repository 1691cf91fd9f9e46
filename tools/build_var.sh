#!/bin/bash
# Build a variant of the CUDA library for A/B timing (tools/ab.sh):
#   bash tools/build_var.sh <name> "<extra nvcc flags>"  -> paper_1209_5421_b200/csrc/build/var/<name>.so
name=$1; extra=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/pkg" "$tmp/out"
cp -r "$root/paper_1209_5421_b200/csrc" "$tmp/pkg/csrc"
cp -r "$root/include" "$tmp/include"
rm -rf "$tmp/pkg/csrc/build"
(cd "$tmp/pkg/csrc" && make -j16 OUT="$tmp/out" NVEXTRA="$extra" "$tmp/out/libauxamg_b200.so" > "$tmp/build.log" 2>&1) || { cat "$tmp/build.log"; exit 1; }
mkdir -p "$root/paper_1209_5421_b200/csrc/build/var"
cp "$tmp/out/libauxamg_b200.so" "$root/paper_1209_5421_b200/csrc/build/var/$name.so"
grep -A2 "${3:-k_bgs_inv}" "$tmp/pkg/csrc/build/${4:-solve}.ptxas.txt" | grep -i "registers\|spill" | head -4
rm -rf "$tmp"
