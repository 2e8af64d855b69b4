export SWB_WATCHDOG_MS=30000
export SWB_LIB=paper_1304_5966_b200/libswb_checked.so
ONLY=85 REPEAT=30 timeout 300 python tools/repro_zero_protein.py "a1" > gpurun_out/g1_chk85.log 2>&1; echo rc=$? >> gpurun_out/g1_chk85.log
timeout 400 python tools/p2_hammer.py 1500 11 > gpurun_out/g1_hchk.log 2>&1; echo rc=$? >> gpurun_out/g1_hchk.log
unset SWB_LIB
ONLY=85 REPEAT=30 timeout 300 python tools/repro_zero_protein.py "a1" > gpurun_out/g1_prod85.log 2>&1; echo rc=$? >> gpurun_out/g1_prod85.log
timeout 400 python tools/repro_zero_protein.py > gpurun_out/g1_prodall.log 2>&1; echo rc=$? >> gpurun_out/g1_prodall.log
timeout 400 python tools/p2_hammer.py 1500 12 > gpurun_out/g1_hprod.log 2>&1; echo rc=$? >> gpurun_out/g1_hprod.log
timeout 600 python tools/narrow_sweep.py protein 300 5 > gpurun_out/g1_nsp.log 2>&1; echo rc=$? >> gpurun_out/g1_nsp.log
timeout 600 python tools/narrow_sweep.py dna 300 6 > gpurun_out/g1_nsd.log 2>&1; echo rc=$? >> gpurun_out/g1_nsd.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.log 2>&1; echo rc=$? >> gpurun_out/g1_tests.log
for f in gpurun_out/g1_*.log; do echo "== $f"; tail -n 2 $f; done
