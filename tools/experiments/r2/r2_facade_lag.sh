#!/bin/bash
out=gpurun_out/facade_lag; mkdir -p $out
for lag in 2 3 4; do
  TSB_ANN_LAG=$lag TSB_FACADE_STATS=1 TSB_FR_CHECKSUM=1 TSB_CONSUMERS=4 timeout 300 python tools/facade_rate.py 4000 > $out/lag_$lag.json 2> $out/lag_$lag.err
  echo "lag $lag $(tail -1 $out/lag_$lag.json) $(grep 'facade stats' $out/lag_$lag.err)"
done | tee $out/summary.txt
