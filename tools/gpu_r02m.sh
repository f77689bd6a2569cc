R=${ROUND_TAG:-r02m}
mkdir -p gpurun_out/$R
timeout 900 python tools/real_rom_families.py 3000 > gpurun_out/$R/families.log 2>&1; echo "rc $?"
