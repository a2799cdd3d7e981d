#!/bin/bash
# Link a variant of libtidas_b200.so with one translation unit recompiled under
# extra -D flags (timing experiments): tools/build_variant.sh <name> <file.cu> <flags...>
# SRC_ROOT=<dir> compiles <dir>/paper_2507_15464_b200/csrc/<file.cu> instead (e.g. a
# `git archive` of an older commit); FTZ=false drops -ftz=true.
set -e
name=$1; src=$2; shift 2
root=${SRC_ROOT:-.}
mkdir -p build/var
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ftz=${FTZ:-true} --expt-relaxed-constexpr"
$NV "$@" -c $root/paper_2507_15464_b200/csrc/$src -o build/var/$name.o
objs=$(ls build/obj/*.o | grep -v "/${src%.cu}.o")
$NV -shared -Xcompiler -fPIC $objs build/var/$name.o -o build/var/lib_$name.so
echo build/var/lib_$name.so
