#!/bin/bash
# Build libmatq.so with extra nvcc flags into build/<name>/ for A/B runs:
#   scripts/build_variant.sh <name> "<-DFLAG=...>"
set -e
cd "$(dirname "$0")/.."
mkdir -p build/$1
make -s -j16 -C paper_2602_03537_b200/csrc EXTRA="$2" OUT=$PWD/build/$1/libmatq.so OBJDIR=$PWD/build/$1/obj 2>&1 | grep -E "error" || true
ls -la build/$1/libmatq.so
