for g in 2 3 5; do
MBX_WIDE_GROUPS=$g timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 4 --csv python tools/probe_step.py --reps 2 2>/dev/null | grep -o '"([0-9]*, [0-9]*, [0-9]*)".*' | awk -F'","' '{print $1, $NF}' | tr -d '"' | tr '\n' ' '; echo
MBX_WIDE_GROUPS=$g MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 1 2>&1 | grep -A4 "cfg 1" | grep "lv  0" | sed 's/\([a-z_0-9]*\) \([-0-9.]*\/[-0-9.]*\)/\n\1 \2/g' | sort -t' ' -k2 -n | tr '\n' ' '; echo
done
