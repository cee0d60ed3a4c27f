mkdir -p gpurun_out/hint
for cfg in "base::" "cs:TSB_CA_ST=cs:" "ldhint:TSB_CA_LDHINT=1:" "both:TSB_CA_ST=cs TSB_CA_LDHINT=1:"; do
  name=${cfg%%:*}; envs=$(echo $cfg | cut -d: -f2)
  for k in f32 bf16; do env $envs timeout 100 python tools/step_floor.py $k host | sed "s/}/, \"cfg\": \"$name\"}/" >> gpurun_out/hint/floor.txt 2>&1; done
done
