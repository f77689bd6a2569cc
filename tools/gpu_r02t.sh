#!/bin/bash
# branch-free epilogue A/B + ping-pong lead sweep
o=gpurun_out/s3; mkdir -p $o
bash tools/ab_libs.sh $o c3:64 "MSW_K1_VARIANT=86 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4" build/ab/lib_base.so build/ab/lib_epi2.so
timeout 300 python tools/variant_bits.py --config c3 --S 64 --steps 64 --variants 69,86,89 > $o/bits.txt 2>&1
cat $o/bits.txt
for lead in 3 4 5 6 8 9; do
  echo "== v 89 lead $lead" >> $o/pp_sweep.log
  MSW_K1_VARIANT=89 MSW_K1_PPLEAD=$lead MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=7,3 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 >> $o/pp_sweep.log 2>&1
done
python - <<'PY'
import json
for f in ("gpurun_out/s3/ab.log", "gpurun_out/s3/pp_sweep.log"):
    for l in open(f):
        if l.startswith('=='): print(l.strip()[:60], end=' ')
        else:
            try:
                d = json.loads(l); print(round(d['ms_step'],4), round(d['k1_ms'],4), d['k1']['k1_variant'], d['k1']['k1_rings'])
            except Exception as e: print('ERR', l[:100])
PY
