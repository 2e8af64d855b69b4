export SWB_WATCHDOG_MS=120000
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
timeout 600 python tools/split_probe.py 1000000 5000000 > gpurun_out/sp5_probe.log 2>&1; echo rc=$? >> gpurun_out/sp5_probe.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-align > gpurun_out/b5.log 2>&1; echo rc=$? >> gpurun_out/b5.log
