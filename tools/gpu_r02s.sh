#!/bin/bash
# round 2 session s: ping-pong consumer groups (variants 89-91) -- parity, bits, timing
mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "fused_layer_kernel" > gpurun_out/s2/fused_tests.log 2>&1
tail -3 gpurun_out/s2/fused_tests.log
timeout 300 python tools/variant_bits.py --config c3 --S 64 --steps 64 --variants 69,86,89,90,91 > gpurun_out/s2/bits.txt 2>&1
cat gpurun_out/s2/bits.txt
for v in 86 89 90 91; do
  for lead in 0 1 2; do
    for rings in 6,4 7,3 5,5; do
      echo "== v $v lead $lead rings $rings" >> gpurun_out/s2/pp_sweep.log
      MSW_K1_VARIANT=$v MSW_K1_PPLEAD=$lead MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=$rings timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 >> gpurun_out/s2/pp_sweep.log 2>&1
    done
    [ $v = 86 ] && break
  done
done
grep -E "==|ms_step" gpurun_out/s2/pp_sweep.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('=='): print(l.strip(), end=' ')
    else:
        try:
            d = json.loads(l); print(round(d['ms_step'],4), round(d['k1_ms'],4), d['k1']['k1_variant'], d['k1']['k1_rings'])
        except Exception as e: print('ERR', l[:100])
"
