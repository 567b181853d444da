#!/bin/bash
# Build libhftw.so from a git revision (default HEAD) into tools/exp/<name>.so for A/B timing
# (HFTW_LIBRARY=tools/exp/<name>.so).  usage: tools/build_variant.sh name [rev|WT] [extra nvcc flags]
# (WT: the working tree)
set -e
name=$1; rev=${2:-HEAD}; shift; shift || true
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
if [ "$rev" = WT ]; then
  mkdir -p "$tmp/paper_1802_05839_b200" && cp -r "$root/paper_1802_05839_b200/csrc" "$tmp/paper_1802_05839_b200/" && cp -r "$root/include" "$tmp/"
else
  git -C "$root" archive "$rev" paper_1802_05839_b200/csrc include | tar -x -C "$tmp"
fi
mkdir -p "$root/tools/exp"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -shared -cudart static "$@" \
  -o "$root/tools/exp/$name.so" "$tmp/paper_1802_05839_b200/csrc/hftw.cu" 2>&1 | grep -E "error" || true
rm -rf "$tmp"
ls -la "$root/tools/exp/$name.so"
