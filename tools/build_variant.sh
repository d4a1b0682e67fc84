#!/bin/bash
# developer: tools/build_variant.sh <name> <extra nvcc flags...>  -> build/variants/lib_<name>.so (reproduce.cu recompiled with the flags)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2404_01159_b200/csrc"
mkdir -p ../../build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC -cudart static "$@" -Xptxas -v -c reproduce.cu -o ../../build/variants/reproduce_$name.o 2> ../../build/variants/reproduce_$name.log
grep -A2 "reproduce_pairs_kernelILi0ELi2" ../../build/variants/reproduce_$name.log | tail -2
objs=$(ls *.o | grep -v reproduce.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../build/variants/lib_$name.so $objs ../../build/variants/reproduce_$name.o
