#!/bin/bash
# time K1 template instances on a config (development aid):
#   tools/variant_sweep.sh <cases> <variant ids...>
cases=${1:-c3:64}; shift
vs=${@:-0 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15}
for v in $vs; do
  MSW_K1_VARIANT=$v python tools/rom_sweep.py --cases $cases --steps 50 2>&1 | sed "s/^/{\"variant\": $v} /"
done
