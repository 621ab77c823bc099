#!/bin/bash
# A/B builds of one kernel file: profiles/ab/build_variant.sh NAME FILE.cu [nvcc flags...]
# -> paper_2403_03605_b200/lib/ab/libpmts_NAME.so (the other objects come from the main build);
# run a variant with PMTS_LIB_PATH=<that file>.
set -e
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/../.." && pwd)
pk=$root/paper_2403_03605_b200
mkdir -p $pk/lib/ab
extra=""
case $src in pd_det.cu|pd_setup.cu|pmts_pd.cu|pd_mts.cu|pmts_mts.cu) extra="-fmad=false";; esac
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v \
  -Xcompiler -fPIC,-ffp-contract=off $extra "$@" -c $pk/csrc/$src -o $pk/lib/ab/$name.$src.o 2> $pk/lib/ab/$name.ptxas.log
objs=""
for o in $pk/lib/obj/*.o; do
  if [ "$(basename $o)" == "$src.o" ]; then objs="$objs $pk/lib/ab/$name.$src.o"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $pk/lib/ab/libpmts_$name.so $objs -lcudart
echo $pk/lib/ab/libpmts_$name.so
