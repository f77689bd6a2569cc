R=${ROUND_TAG:-r02i}
mkdir -p gpurun_out/$R
for dbg in 8 9; do
  echo "dbg=$dbg" >> gpurun_out/$R/prof.log
  MSW_LIB=build/prof/libmswave_b200.so MSW_K1_DEBUG=$dbg MSW_K1_VARIANT=69 MSW_K1_RINGS=6,4 MSW_K1_FUSED_UPG=0 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 100 >> gpurun_out/$R/prof.log 2>&1
done
