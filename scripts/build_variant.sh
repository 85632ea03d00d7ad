#!/bin/bash
# Build the product library with extra nvcc flags into exp/<name>.so
# (development aid for A/B timing), then restore the default build.
# usage: scripts/build_variant.sh <name> "<EXTRA flags>"
set -e
cd "$(dirname "$0")/../paper_1606_06659_b200/csrc"
make clean >/dev/null
make EXTRA="$2" >/dev/null 2>&1 || { make EXTRA="$2" 2>&1 | tail -20; exit 1; }
mkdir -p ../../exp
cp ../lib/libcountmc_b200.so ../../exp/$1.so
grep -A2 "eps_sweep_kernel\|gene_sweep_kernel" ../lib/sweep_kernels.ptxas.txt | grep -E "registers|spill" | sed "s/^/$1: /"
make clean >/dev/null
make >/dev/null 2>&1
