#!/bin/bash
# Build the library from a source tree (default: this repo) into paper_1808_01517_b200/libdelimit_<tag>.so
# for A/B timing on one GPU box:  DELIMIT_LIB=paper_1808_01517_b200/libdelimit_<tag>.so python bench.py ...
# usage: scripts/build_variant.sh <tag> [src_root] [extra nvcc flags...]
set -e
root=$(cd $(dirname $0)/.. && pwd)
tag=$1; src=${2:-$root}; shift; shift || true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -I $src/include "$@" -o $root/paper_1808_01517_b200/libdelimit_$tag.so \
  $src/paper_1808_01517_b200/csrc/*.cu
