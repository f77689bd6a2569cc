R=r02a
mkdir -p gpurun_out/$R
nvidia-smi -q | grep -i -A3 "clocks" | head -20 > gpurun_out/$R/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
timeout 600 python bench.py > gpurun_out/$R/bench_c3.json 2> gpurun_out/$R/bench_c3.err; echo "bench rc $?"
