# round-end evidence: bench line (config 3 + config-5 sweep + real ROM +
# full-length e2e), reference arm, ncu launch list of the bench command and
# full captures of the top kernels
R=${ROUND_TAG:-r02final}
mkdir -p gpurun_out/$R
# the bench run tunes each shape once and records it; the ncu runs below then
# reuse the tuned geometry (their launch lists hold no tuning launches)
export MSW_TUNE_CACHE=$PWD/gpurun_out/$R/tune_cache.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/$R/smi.txt 2>&1
timeout 1200 python bench.py > gpurun_out/$R/bench_c3.json 2> gpurun_out/$R/bench_c3.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/$R/bench_ref.json 2> gpurun_out/$R/bench_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$R/launches_bench_c3.csv python bench.py --steps 20 --warmup 3 --no-fine --no-cpu --no-sweep > gpurun_out/$R/ncu_launch.log 2>&1; echo "ncu launch rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rom_cell_fused|rom_iface_step" -s 6 -c 2 -o gpurun_out/$R/full_c3 python tools/rom_sweep.py --cases c3:64 --steps 5 > gpurun_out/$R/ncu_full_c3.log 2>&1; echo "ncu c3 rc $?"
timeout 900 ncu --set full --clock-control none -k regex:"rom_cell_kstream" -s 3 -c 1 -o gpurun_out/$R/full_c5s128 python tools/rom_sweep.py --cases c5:128 --steps 5 > gpurun_out/$R/ncu_full_c5s128.log 2>&1; echo "ncu c5 rc $?"
timeout 900 ncu --set full --clock-control none -k regex:"fine_zmarch" -s 2 -c 1 -o gpurun_out/$R/full_fine_c3 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep > gpurun_out/$R/ncu_full_fine.log 2>&1; echo "ncu fine rc $?"
