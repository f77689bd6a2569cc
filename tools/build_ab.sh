#!/bin/bash
# A/B library builds: build_ab.sh NAME [extra nvcc flags...] -> build/ab/lib_NAME.so
# (load with MSW_LIB=...; tools/ab_libs.sh times several builds interleaved)
set -e
name=$1; shift
d=$(dirname "$0")/../paper_1604_06750_b200/csrc
o=$(dirname "$0")/../build/ab; mkdir -p $o/obj_$name
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in rom_system fine_system; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c -o $o/obj_$name/$f.o $d/$f.cu &
done
for f in mswave_api rom_archive; do
  nvcc $ARCH -std=c++17 -O2 -I$d/../../include -Xcompiler -fPIC -Xcompiler -ffp-contract=off -c -o $o/obj_$name/$f.o $d/$f.cpp &
done
wait
nvcc $ARCH -shared -o $o/lib_$name.so $o/obj_$name/*.o -lcudart
echo built $o/lib_$name.so
