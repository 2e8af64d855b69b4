export SWB_WATCHDOG_MS=120000
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
timeout 600 python tools/option_ab.py 5000000 x2 1 2 > gpurun_out/c3_6.log 2>&1
