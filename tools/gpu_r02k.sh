R=${ROUND_TAG:-r02k}
mkdir -p gpurun_out/$R
echo "c3 S=1 tuned (prof build)" >> gpurun_out/$R/prof.log
MSW_LIB=build/prof/libmswave_b200.so MSW_K1_DEBUG=8 MSW_K1_TUNE_LOG=1 timeout 300 python tools/rom_sweep.py --cases c3:1 --steps 200 >> gpurun_out/$R/prof.log 2>&1
for v in 69 73 74 75 76; do
  echo "variant=$v" >> gpurun_out/$R/prof.log
  MSW_LIB=build/prof/libmswave_b200.so MSW_K1_DEBUG=8 MSW_K1_VARIANT=$v timeout 300 python tools/rom_sweep.py --cases c3:1 --steps 200 >> gpurun_out/$R/prof.log 2>&1
done
