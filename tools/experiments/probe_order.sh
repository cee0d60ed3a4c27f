mkdir -p gpurun_out/ord
o=gpurun_out/ord/sweep.txt
for ord in rr blocked; do
 for occ in 0 2 3 4; do
  echo "order=$ord occ=$occ" >> $o
  TSB_CA_ORDER=$ord TSB_CA_OCC=$occ timeout 300 python tools/sweep_collate.py 4,8,16 2,3 >> $o 2>&1
 done
done
