# A/B of a compile-time variant: ncu kernel durations of the levels launches with and without $1=1
mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export $1=1; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 12 --csv --log-file gpurun_out/ab_$v.csv python tools/probe_step.py --reps 4 > /dev/null 2>&1
  echo "variant $v"; grep -o '"(1, 16, 8)".*' gpurun_out/ab_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
done
