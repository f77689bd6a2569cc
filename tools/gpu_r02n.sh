R=${ROUND_TAG:-r02n}
mkdir -p gpurun_out/$R
timeout 600 python tools/rom_sweep.py --cases c3:64,c2:16,c1:1 --steps 100 > gpurun_out/$R/sweep.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s -k "real_rom or fused or every_k1 or config1 or config2" > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
