#!/bin/bash
o=gpurun_out/s4; mkdir -p $o
MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=8 MSW_K1_VARIANT=86 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 > $o/prof86.log 2>&1
cat $o/prof86.log | cut -c1-400
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "fused" > $o/fused_tests.log 2>&1
tail -3 $o/fused_tests.log
