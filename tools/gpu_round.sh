SWB_WATCHDOG_MS=60000 timeout 900 python -m pytest tests/test_gpu_scale_golden.py -q -x -k "concurrent or slabs" > gpurun_out/sg2.log 2>&1; echo rc=$? >> gpurun_out/sg2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/b2.log 2>&1; echo rc=$? >> gpurun_out/b2.log
