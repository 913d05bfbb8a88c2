# A/B: levels launch durations (ncu) with $1 unset vs set to $2
mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export $1=$2; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 12 --csv --log-file gpurun_out/ab_$v.csv python tools/probe_step.py --reps 4 > gpurun_out/ab_$v.log 2>&1
  echo "variant $v"; grep -o '"([0-9]*, [0-9]*, [0-9]*)".*' gpurun_out/ab_$v.csv | awk -F'","' '{print $1, $NF}' | tr -d '"' | tr '\n' ' '; echo
done
