mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:plan_vm_kernel --launch-skip 20 --launch-count 1 -o gpurun_out/vm_full -f python tools/probe_step.py --model nestedrnn --reps 1 > gpurun_out/vm_full.log 2>&1
tail -2 gpurun_out/vm_full.log
