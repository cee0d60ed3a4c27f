mkdir -p gpurun_out/p11
timeout 200 python tools/dbg_rebatch.py > gpurun_out/p11/dbg.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -o faulthandler_timeout=200 > gpurun_out/p11/all.log 2>&1; echo "rc=$?" >> gpurun_out/p11/all.log
