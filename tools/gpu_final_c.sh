#!/bin/bash
# round-end evidence, final code of round 2: full GPU test suite, then tools/gpu_final.sh
# (bench line, reference arm, ncu launch list and full captures), plus a config-5 S=32 capture
export ROUND_TAG=final_c
mkdir -p gpurun_out/$ROUND_TAG
timeout 3000 python -m pytest tests -x -q -m gpu > gpurun_out/$ROUND_TAG/gpu_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/$ROUND_TAG/gpu_tests.log
bash tools/gpu_final.sh
export MSW_TUNE_CACHE=$PWD/gpurun_out/$ROUND_TAG/tune_cache.txt
timeout 900 ncu --set full --clock-control none -k regex:"rom_cell_kstream" -s 3 -c 1 -o gpurun_out/$ROUND_TAG/full_c5s32 python tools/rom_sweep.py --cases c5:32 --steps 5 > gpurun_out/$ROUND_TAG/ncu_full_c5s32.log 2>&1; echo "ncu c5s32 rc $?"
python tools/ncu_summary.py gpurun_out/$ROUND_TAG/full_c3.ncu-rep gpurun_out/$ROUND_TAG/full_c5s128.ncu-rep gpurun_out/$ROUND_TAG/full_c5s32.ncu-rep gpurun_out/$ROUND_TAG/full_fine_c3.ncu-rep > gpurun_out/$ROUND_TAG/ncu_summary.json 2> gpurun_out/$ROUND_TAG/ncu_summary.err
# the reports (source import) are too large to bring back; the summaries above hold what DESIGN cites
for r in full_c3 full_c5s128 full_c5s32 full_fine_c3; do ncu -i gpurun_out/$ROUND_TAG/$r.ncu-rep --page raw --csv > gpurun_out/$ROUND_TAG/$r.raw.csv 2>/dev/null; rm -f gpurun_out/$ROUND_TAG/$r.ncu-rep; done
du -sh gpurun_out/$ROUND_TAG
python __graft_entry__.py smoke > gpurun_out/$ROUND_TAG/smoke.log 2>&1; tail -1 gpurun_out/$ROUND_TAG/smoke.log
cat gpurun_out/$ROUND_TAG/bench_c3.json | cut -c1-600
