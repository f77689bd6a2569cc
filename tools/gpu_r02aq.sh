#!/bin/bash
# final check of the last K2 change: ROM / config / real-ROM / diag parity, then the bench line
o=gpurun_out/aq; mkdir -p $o
timeout 2400 python -m pytest tests -x -q -m gpu > $o/gpu_tests.log 2>&1; echo "tests rc $?"; tail -3 $o/gpu_tests.log
export MSW_TUNE_CACHE=$PWD/$o/tune_cache.txt
timeout 1200 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err; echo "bench rc $?"
python - <<'PY'
import json
d=json.load(open("gpurun_out/aq/bench_c3.json"))
print('c3', d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline']['iface_kernel_ms'], d['roofline']['step']['frac'], d['clocks']['sm_mhz'], 'e2e', d['e2e']['value'])
for k,p in d['sweep']['c5']['points'].items():
    print(k, round(p['ms_per_step'],4), round(p['step_hbm_frac'],3), round(p['step_fp64_frac'],3), round(p['k1_in_step_ms'],4), round(p['k2_alone_ms'],4), '%.3g'%p['e2e']['value'], p['k1']['k1_variant'])
PY
