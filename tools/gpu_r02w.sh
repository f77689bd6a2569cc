#!/bin/bash
o=gpurun_out/s8; mkdir -p $o
for v in 86 89; do for dbg in 8 12 10; do
echo "== v $v dbg $dbg" >> $o/prof.log
MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=$dbg MSW_K1_VARIANT=$v MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 2>&1 | cut -c1-120 >> $o/prof.log
done; done
cat $o/prof.log
