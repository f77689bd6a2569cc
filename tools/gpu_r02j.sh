R=${ROUND_TAG:-r02j}
mkdir -p gpurun_out/$R
for st in 0 1500 3000 4500 6000 9000; do
  echo "stagger=$st" >> gpurun_out/$R/ab.log
  MSW_K1_STAGGER=$st MSW_K1_VARIANT=69 MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 >> gpurun_out/$R/ab.log 2>&1
done
