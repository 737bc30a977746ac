python scripts/one_call.py 21 > /dev/null
for lb in 8 16 32; do TC_LB=$lb ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_rs_pass --csv python scripts/one_call.py 21 2>/dev/null | grep k_rs_pass | awk -F'","' -v lb=$lb '{gsub(/"/,"",$NF); s+=$NF; n++} END {print "lb", lb, n, s/1e3, "us"}'; done
for lb in 8 16 32; do TC_LB=$lb python scripts/probe_s21.py 21 "[{}]" | tail -1; done
