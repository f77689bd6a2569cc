#!/bin/bash
o=gpurun_out/dbg; mkdir -p $o
MSW_K1_FUSED=1 MSW_K1_VARIANT=${V:-69} timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/variant_bits.py --config c2 --S 16 --steps 4 --variants ${V:-69} > $o/memcheck.log 2>&1
grep -v "^=========     at\|^=========         in\|Host Frame\|^=========$" $o/memcheck.log | head -40
