R=${ROUND_TAG:-r02g}
mkdir -p gpurun_out/$R
MSW_K1_VARIANT=86 MSW_K1_RINGS=6,4 timeout 900 ncu --set full --import-source on --clock-control none -k regex:rom_cell_fused -s 6 -c 1 -o gpurun_out/$R/full_c3_k1_ifuse python tools/rom_sweep.py --cases c3:64 --steps 5 > gpurun_out/$R/ncu.log 2>&1; echo "ncu rc $?"
