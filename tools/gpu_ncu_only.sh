mkdir -p gpurun_out
t() { echo "== $*"; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 4 --csv python tools/probe_step.py --reps 2 2>&1 | grep -i "error\|mbx_tc_levels" | cut -c1-160 | head -6; }
t X=1
t MBX_NO_COOP=1
t MBX_LEVELS_WIDE=4,128
t MBX_LEVELS_WIDE=4,128 MBX_NO_COOP=1
t MBX_ARRIVE_RELEASE=1
