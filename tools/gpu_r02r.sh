R=${ROUND_TAG:-r02r}
mkdir -p gpurun_out/$R
./tools/probe/fp64_peak dmma > gpurun_out/$R/fp64_probe.txt 2>&1
timeout 900 python bench.py --steps 100 --no-cpu > gpurun_out/$R/bench.json 2> gpurun_out/$R/bench.err; echo "bench rc $?"
