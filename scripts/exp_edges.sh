python scripts/one_call.py 21 > /dev/null
for e in 0 1 2 4 7; do TC_EXP=$e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k k_edges --csv python scripts/one_call.py 21 2>/dev/null | grep k_edges | awk -F'","' -v e=$e '{print "exp", e, $(NF-2), $(NF-1), $NF}'; done
