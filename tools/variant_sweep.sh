#!/bin/bash
# time every K1 template instance that fits a config (development aid)
for v in 0 1 2 3 4 5 6 7 8 9; do
  MSW_K1_VARIANT=$v python tools/rom_sweep.py --cases ${1:-c3:64} --steps 50 2>&1 | sed "s/^/{\"variant\": $v} /"
done
