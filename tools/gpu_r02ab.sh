#!/bin/bash
# config 5 S = 32 / 128: where the K-streaming cell kernel's time goes
o=gpurun_out/ab; mkdir -p $o
export MSW_TUNE_CACHE=$PWD/$o/tune_cache.txt
MSW_K1_TUNE_LOG=1 timeout 600 python tools/rom_sweep.py --cases c5:32,c5:128 --steps 30 > $o/base.log 2> $o/tune.log
MSW_K1_DEBUG=1 timeout 600 python tools/rom_sweep.py --cases c5:32,c5:128 --steps 30 > $o/skipmath.log 2>&1
MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=8 timeout 600 python tools/rom_sweep.py --cases c5:32 --steps 30 > $o/prof32.log 2>&1
MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=8 timeout 600 python tools/rom_sweep.py --cases c5:128 --steps 30 > $o/prof128.log 2>&1
cat $o/tune_cache.txt
for f in base skipmath prof32 prof128; do echo "== $f"; cut -c1-330 $o/$f.log | tail -4; done
