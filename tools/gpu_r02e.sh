R=${ROUND_TAG:-r02e}
mkdir -p gpurun_out/$R
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_configs_gpu.py > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
for v in 69 86; do
  echo "variant=$v" >> gpurun_out/$R/ab.log
  MSW_K1_VARIANT=$v MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64,c3:1,c2:16 --steps 200 >> gpurun_out/$R/ab.log 2>&1
done
echo "autotuned" >> gpurun_out/$R/ab.log
MSW_K1_TUNE_LOG=1 timeout 300 python tools/rom_sweep.py --cases c3:64,c2:16,c1:1 --steps 200 >> gpurun_out/$R/ab.log 2>&1
