mkdir -p gpurun_out
MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 2 > gpurun_out/stamps_nopdl.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_small -c 8 --csv --log-file gpurun_out/small_bf.csv python tools/probe_step.py --reps 2 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
