# A/B/C: levels launch durations (ncu) for env $1 over values $2..; plus levels parity test
mkdir -p gpurun_out
var=$1; shift
for v in "$@"; do
  export $var=$v
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 12 --csv --log-file gpurun_out/ab_$v.csv python tools/probe_step.py --reps 4 > gpurun_out/ab_$v.log 2>&1
  echo "$var=$v"; grep -o '"([0-9]*, [0-9]*, [0-9]*)".*' gpurun_out/ab_$v.csv | awk -F'","' '{print $1, $NF}' | tr -d '"' | tr '\n' ' '; echo
done
unset $var
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "levels or baseline" 2>&1 | tail -3
