R=${ROUND_TAG:-r02h}
mkdir -p gpurun_out/$R
for upg in 0 1; do
 for rings in 6,4 7,3 5,5 8,3 6,5 5,6; do
  echo "upg=$upg rings=$rings" >> gpurun_out/$R/ab.log
  MSW_K1_FUSED_UPG=$upg MSW_K1_VARIANT=69 MSW_K1_RINGS=$rings timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 >> gpurun_out/$R/ab.log 2>&1
 done
done
MSW_K1_FUSED_UPG=1 timeout 300 python tools/rom_sweep.py --cases c3:64,c3:1,c2:16,c1:1 --steps 200 >> gpurun_out/$R/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fused or fullsize" > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
