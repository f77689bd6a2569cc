run() { env "$@" python tools/rom_sweep.py --cases c5:8 --steps 30 2>&1 | sed "s/^/{\"env\": \"$*\"} /"; }
run X=0
run MSW_K1_DEBUG=16
run MSW_K1_NP=32
run MSW_K1_NP=32 MSW_K1_DEBUG=16
run MSW_K1_NP=16
run MSW_K1_NP=16 MSW_K1_DEBUG=16
run MSW_K1_NP=104
run MSW_K1_VARIANT=4 MSW_K1_NP=32
run MSW_K1_VARIANT=6 MSW_K1_NP=16
