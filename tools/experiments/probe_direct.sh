mkdir -p gpurun_out/dir
TSB_CA_IMPL=direct timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_group.py -q -x > gpurun_out/dir/pytest.log 2>&1
for impl in tma direct; do
  for k in f32 bf16 u8; do TSB_CA_IMPL=$impl timeout 100 python tools/step_floor.py $k graph | sed "s/}/, \"impl\": \"$impl\"}/" >> gpurun_out/dir/floor.txt 2>&1; TSB_CA_IMPL=$impl timeout 100 python tools/step_floor.py $k host | sed "s/}/, \"impl\": \"$impl\"}/" >> gpurun_out/dir/floor.txt 2>&1; done
done
