SWB_WATCHDOG_MS=60000 timeout 900 python -m pytest tests/test_gpu_scale_golden.py -q -x -k "concurrent or slabs or shared" > gpurun_out/sg3.log 2>&1; echo rc=$? >> gpurun_out/sg3.log
