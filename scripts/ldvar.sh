for v in ${@:-head reg0 reg1}; do
  TC_LIB=$PWD/variants/$v/libtc_b200.so timeout 300 python scripts/probe_lowdeg.py road 2>&1 | grep lowdeg
  TC_LIB=$PWD/variants/$v/libtc_b200.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ld_launches_$v.csv python scripts/one_lowdeg.py > /dev/null 2>&1
  echo "== $v"; python scripts/launch_table.py gpurun_out/ld_launches_$v.csv 2>&1 | head -9
done
