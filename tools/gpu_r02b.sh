R=${ROUND_TAG:-r02b}
mkdir -p gpurun_out/$R
nproc > gpurun_out/$R/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
timeout 900 python bench.py > gpurun_out/$R/bench_c3.json 2> gpurun_out/$R/bench_c3.err; echo "bench rc $?"
