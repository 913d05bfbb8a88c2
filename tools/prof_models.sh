# ncu launch lists (kernel, grid, duration, DRAM bytes) of one mini-batch of every BASELINE config,
# in the product issue order (--plain: no per-batch timing events).
mkdir -p gpurun_out
L="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 300 ncu $L --log-file gpurun_out/launches_treelstm512_b64.csv python tools/probe_step.py --reps 2 --plain > /dev/null 2>&1
timeout 300 ncu $L --log-file gpurun_out/launches_treelstm256_b8.csv python tools/probe_step.py --model treelstm --hidden 256 --batch 8 --precision fp32 --reps 2 --plain > /dev/null 2>&1
timeout 300 ncu $L --log-file gpurun_out/launches_birnn512_b64.csv python tools/probe_step.py --model birnn --hidden 512 --batch 64 --reps 2 --plain > /dev/null 2>&1
timeout 300 ncu $L --log-file gpurun_out/launches_mvrnn128_b64.csv python tools/probe_step.py --model mvrnn --hidden 128 --batch 64 --precision fp32 --reps 2 --plain > /dev/null 2>&1
timeout 600 ncu $L --log-file gpurun_out/launches_nestedrnn512_b64.csv python tools/probe_step.py --model nestedrnn --hidden 512 --batch 64 --reps 1 --plain > /dev/null 2>&1
for f in gpurun_out/launches_*.csv; do echo "$f $(python tools/ncu_list.py $f | wc -l) launches, $(python tools/ncu_list.py $f | awk '{s+=$(NF-2)} END {print s}') us"; done
