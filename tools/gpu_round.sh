export SWB_WATCHDOG_MS=120000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_golden.py -q -x -k "groups or split" > gpurun_out/f1s.log 2>&1; echo rc=$? >> gpurun_out/f1s.log
