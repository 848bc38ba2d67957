#!/bin/bash
# per-kernel launch list of one C3 LTTB call (n_out 1000 and 10000) under ncu
for n in 1000 10000; do
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/lttb_launches_$n.csv \
      python tools/profile_lttb.py $n 2 > gpurun_out/ncu_l_$n.log 2>&1
done
