mkdir -p gpurun_out/ord2
o=gpurun_out/ord2/sweep.txt
for rep in 1 2; do
for cfg in 1:16:3 1:16:4 1:8:6 1:32:2 2:8:3 2:8:4 2:16:2 2:4:6 3:8:2 3:4:4 0:4:3; do
  IFS=: read occ r st <<< "$cfg"
  echo -n "occ=$occ " >> $o
  TSB_CA_OCC=$occ timeout 200 python tools/sweep_collate.py $r $st >> $o 2>&1
done
done
