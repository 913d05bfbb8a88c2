# A/B: wide-config levels launch (first mbx_tc_levels of a step) under env $1 = each of $2..
mkdir -p gpurun_out
var=$1; shift
for v in "$@"; do
  if [ "$v" = none ]; then unset $var; else export $var=$v; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 8 --csv --log-file gpurun_out/ab_w.csv python tools/probe_step.py --reps 2 > gpurun_out/ab_w.log 2>&1
  echo "$var=$v"; grep -o '"([0-9]*, [0-9]*, [0-9]*)".*' gpurun_out/ab_w.csv | awk -F'","' '{print $1, $NF}' | tr -d '"' | tr '\n' ' '; echo
  MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 1 2>&1 | grep -A3 "cfg 1" | head -4 | cut -c1-400
done
