R=${ROUND_TAG:-r02q}
mkdir -p gpurun_out/$R
for i in 1 2; do
  echo "r01 build" >> gpurun_out/$R/fine_ab.log
  (cd build/r1src && timeout 600 python tools/fine_sweep.py --cases c3:64,c3:1,c5:8,c5:32 --steps 10) >> gpurun_out/$R/fine_ab.log 2>&1
  echo "current build" >> gpurun_out/$R/fine_ab.log
  timeout 600 python tools/fine_sweep.py --cases c3:64,c3:1,c5:8,c5:32 --steps 10 >> gpurun_out/$R/fine_ab.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fine" > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
