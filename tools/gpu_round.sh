export SWB_WATCHDOG_MS=120000
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
