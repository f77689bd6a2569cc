R=${ROUND_TAG:-r02c}
mkdir -p gpurun_out/$R
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k1_loop_probe k1_loop_probe.cu && timeout 300 ./k1_loop_probe > ../../gpurun_out/$R/k1_loop_probe.txt 2>&1; cd ../..
echo "probe rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rom_cell_fused -s 6 -c 1 -o gpurun_out/$R/full_c3_k1 python tools/rom_sweep.py --cases c3:64 --steps 5 > gpurun_out/$R/ncu_c3.log 2>&1; echo "ncu rc $?"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_configs_gpu.py > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
