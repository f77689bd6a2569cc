R=${ROUND_TAG:-r02p}
mkdir -p gpurun_out/$R
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
ROUND_TAG=r02b_final bash tools/gpu_final.sh
