out=gpurun_out/san_pt; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 --error-exitcode 9 \
      python -m pytest tests/test_gpu_pipeline.py -q -x -p no:cacheprovider -k "persistent or ingest" > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/summary.txt
done
cat $out/summary.txt
