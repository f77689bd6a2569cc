for d in 0 16 32 64 112; do
  MSW_K1_DEBUG=$d python tools/rom_sweep.py --cases c3:64 --steps 50 2>&1 | sed "s/^/{\"dbg\": $d} /"
done
