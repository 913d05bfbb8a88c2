mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/nested_launches.csv python tools/probe_step.py --model nestedrnn --reps 1 > gpurun_out/nested_probe.log 2>&1
tail -3 gpurun_out/nested_probe.log
