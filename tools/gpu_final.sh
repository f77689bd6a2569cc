# round-end evidence: tests, bench lines (c3 default + c5 sweep), reference arm,
# ncu launch list of the bench command and full captures of the top kernels
set -x
R=${ROUND_TAG:-r01g}
mkdir -p gpurun_out/$R
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$R/gpu_tests.log 2>&1; echo "tests rc $?"
timeout 900 python bench.py > gpurun_out/$R/bench_c3.json 2> gpurun_out/$R/bench_c3.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/$R/bench_ref.json 2> gpurun_out/$R/bench_ref.err; echo "ref rc $?"
for S in 1 8 32 128; do
  timeout 900 python bench.py --config c5 --sources $S --steps 100 > gpurun_out/$R/bench_c5s$S.json 2> gpurun_out/$R/bench_c5s$S.err; echo "c5 S=$S rc $?"
done
for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 200 > gpurun_out/$R/bench_$c.json 2> gpurun_out/$R/bench_$c.err; echo "$c rc $?"
done
MSW_K1_VARIANT=69 MSW_K1_RINGS=7,3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/$R/launches_bench_c3.csv python bench.py --steps 20 --warmup 3 --no-fine --no-cpu > gpurun_out/$R/ncu_launch.log 2>&1; echo "ncu launch rc $?"
MSW_K1_VARIANT=69 MSW_K1_RINGS=7,3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rom_cell_fused|rom_iface_step" -s 6 -c 2 -o gpurun_out/$R/full_c3 python tools/rom_sweep.py --cases c3:64 --steps 5 > gpurun_out/$R/ncu_full_c3.log 2>&1; echo "ncu c3 rc $?"
MSW_K1_VARIANT=36 MSW_K1_NP=64 MSW_K1_RINGS=3,3 timeout 900 ncu --set full --clock-control none -k regex:rom_cell_kstream -s 3 -c 1 -o gpurun_out/$R/full_c5s8 python tools/rom_sweep.py --cases c5:8 --steps 5 > gpurun_out/$R/ncu_full_c5s8.log 2>&1; echo "ncu c5s8 rc $?"
MSW_K1_VARIANT=32 MSW_K1_NP=64 MSW_K1_RINGS=2,2 timeout 900 ncu --set full --clock-control none -k regex:rom_cell_kstream -s 3 -c 1 -o gpurun_out/$R/full_c5s32 python tools/rom_sweep.py --cases c5:32 --steps 5 > gpurun_out/$R/ncu_full_c5s32.log 2>&1; echo "ncu c5s32 rc $?"
