R=${ROUND_TAG:-r02d}
mkdir -p gpurun_out/$R
for dbg in 0 32 1 33; do
  echo "dbg=$dbg" >> gpurun_out/$R/ab.log
  MSW_K1_VARIANT=69 MSW_K1_RINGS=6,4 MSW_K1_DEBUG=$dbg timeout 300 python tools/rom_sweep.py --cases c3:64,c3:1 --steps 200 >> gpurun_out/$R/ab.log 2>&1
done
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_configs_gpu.py > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
