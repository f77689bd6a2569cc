#!/bin/bash
# the driver's likely invocations, timed by wall clock
o=gpurun_out/ar; mkdir -p $o
t0=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 3 > $o/bench_20.json 2> $o/bench_20.err; echo "bench rc $? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 3 > $o/ref_20.json 2> $o/ref_20.err; echo "ref rc $? wall $(( $(date +%s) - t0 )) s"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/ar/bench_20.json").read().strip().splitlines()[-1])
print(sorted(d.keys()))
print(d['ms_per_step'], d['value'], d['steps'], d['warmup'], d['gpu_launches'], d['roofline']['frac'], d['roofline']['step']['frac'], d['clocks'])
r=json.loads(open("gpurun_out/ar/ref_20.json").read().strip().splitlines()[-1])
print(r['impl'], r['value'], r['ms_per_step'], r['config']['sources_per_gpu'], r['cpu_baseline'])
PY
