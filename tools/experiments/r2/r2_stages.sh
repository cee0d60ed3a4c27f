#!/bin/bash
# fused checksum kernel: rows per item x item stages
out=gpurun_out/${1:-stg}; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_crc_fused.py -q -x > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for cfg in "32 8" "32 2" "16 8" "16 4" "16 3" "8 8"; do set -- $cfg
  TSB_CA_R=$1 TSB_CC_STAGES=$2 timeout 300 python tools/crc_fused_timing.py f32,bf16 200 | grep '"checksum": true' | sed "s/^{/{\"R\": $1, \"stages_cap\": $2, /" >> $out/timing.jsonl 2>> $out/timing.err
done
