#!/bin/bash
o=gpurun_out/s11; mkdir -p $o
bash tools/ab_libs.sh $o c3:64,c2:16 "MSW_K1_FUSED=0 MSW_TUNE_FRESH=1" build/ab/lib_base.so build/ab/lib_pipe2.so
python - <<'PY'
import json
for l in open("gpurun_out/s11/ab.log"):
    if l.startswith('=='): print(l.strip()[:70])
    else:
        try:
            d = json.loads(l); print(d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_rings'])
        except Exception as e: print('ERR', l[:100])
PY
timeout 2400 python -m pytest tests -x -q -m gpu > $o/gpu_tests.log 2>&1
tail -3 $o/gpu_tests.log
