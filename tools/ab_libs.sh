#!/bin/bash
# A/B device timing of library builds: ab_libs.sh OUTDIR CASES "ENV" LIB1 LIB2 ...
# Each lib is timed twice, interleaved, with the same pinned K1 env (rom_sweep.py).
out=$1; cases=$2; envs=$3; shift 3
mkdir -p "$out"
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib rep $rep env [$envs]" >> "$out/ab.log"
    env $envs MSW_LIB=$(realpath "$lib") timeout 600 python tools/rom_sweep.py --cases "$cases" --steps 200 >> "$out/ab.log" 2>> "$out/ab.err"
  done
done
