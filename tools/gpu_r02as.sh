#!/bin/bash
# ncu full captures of the config-3 kernels with the final code (K2 at 96 threads, loads before the barrier)
o=gpurun_out/as; mkdir -p $o
export MSW_TUNE_CACHE=$PWD/$o/tune_cache.txt
timeout 600 python tools/rom_sweep.py --cases c3:64 --steps 50 > $o/sweep.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rom_cell_fused|rom_iface_step" -s 6 -c 2 -o $o/full_c3 python tools/rom_sweep.py --cases c3:64 --steps 5 > $o/ncu_full_c3.log 2>&1; echo "ncu c3 rc $?"
python tools/ncu_summary.py $o/full_c3.ncu-rep > $o/ncu_summary_c3.json 2> $o/ncu_summary.err
ncu -i $o/full_c3.ncu-rep --page raw --csv > $o/full_c3.raw.csv 2>/dev/null
ncu -i $o/full_c3.ncu-rep --page source --csv -k regex:"rom_cell_fused" > $o/full_c3_k1.source.csv 2>/dev/null; ls -la $o
rm -f $o/full_c3.ncu-rep
cut -c1-400 $o/sweep.log | tail -1
