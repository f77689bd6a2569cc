R=${ROUND_TAG:-r02o}
mkdir -p gpurun_out/$R
for i in 1 2 3; do
  echo "r01 build" >> gpurun_out/$R/ab.log
  (cd build/r1src && MSW_K1_VARIANT=69 MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 400) >> gpurun_out/$R/ab.log 2>&1
  echo "current build" >> gpurun_out/$R/ab.log
  MSW_K1_VARIANT=69 MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 400 >> gpurun_out/$R/ab.log 2>&1
done
