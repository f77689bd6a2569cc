#!/bin/bash
o=gpurun_out/ao; mkdir -p $o
timeout 1800 python -m pytest tests/test_rom_gpu.py tests/test_configs_gpu.py -x -q -m gpu > $o/rom.log 2>&1; tail -3 $o/rom.log
