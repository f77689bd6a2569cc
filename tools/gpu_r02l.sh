R=${ROUND_TAG:-r02l}
mkdir -p gpurun_out/$R
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s -k "real_rom" > gpurun_out/$R/real_rom.log 2>&1; echo "real rc $?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
