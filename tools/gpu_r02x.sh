#!/bin/bash
o=gpurun_out/s7; mkdir -p $o
MSW_LIB=$(realpath build/ab/lib_base.so) timeout 300 python tools/variant_bits.py --config c3 --S 64 --steps 64 --variants 69,86 > $o/bits_base.txt 2>&1
timeout 300 python tools/variant_bits.py --config c3 --S 64 --steps 64 --variants 69,86,89,90,92 > $o/bits.txt 2>&1
cat $o/bits_base.txt $o/bits.txt | cut -c1-200
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "fused" > $o/fused_tests.log 2>&1
tail -3 $o/fused_tests.log
bash tools/ab_libs.sh $o c3:64 "MSW_K1_VARIANT=86 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4" build/ab/lib_epi2.so build/ab/lib_perm.so
bash tools/ab_libs.sh $o c3:64 "MSW_K1_VARIANT=89 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4" build/ab/lib_perm.so
bash tools/ab_libs.sh $o c3:64 "MSW_K1_VARIANT=90 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4" build/ab/lib_perm.so
bash tools/ab_libs.sh $o c3:64 "MSW_K1_VARIANT=87 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4" build/ab/lib_perm.so
python - <<'PY'
import json
for l in open("gpurun_out/s7/ab.log"):
    if l.startswith('=='): print(l.strip()[:70], end=' ')
    else:
        try:
            d = json.loads(l); print(round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_rings'])
        except Exception as e: print('ERR', l[:100])
PY
