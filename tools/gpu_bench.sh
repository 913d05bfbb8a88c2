# Bench + launch list + ncu of the dominant kernel; results under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mbx_tc_levels --launch-skip 3 --launch-count 1 -o gpurun_out/levels_full -f python tools/probe_step.py --reps 5 > gpurun_out/ncu_levels.log 2>&1
tail -1 gpurun_out/bench.log
