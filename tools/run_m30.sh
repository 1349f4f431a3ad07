# The bounds-checked build (RII_LIB=checked) at the final sources: whole GPU suite, then the M = 8
# suites with either thread count forced, and the checked sanitizer drive.
set -x
T=${TAG:-r02t}
RII_LIB=checked timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest_gpu_$T.log 2>&1; echo checked=$?
RII_LIB=checked RII_M8_NTH=384 timeout 900 python -m pytest tests/test_gpu_windows.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/checked_pytest_m8nth384_$T.log 2>&1; echo c384=$?
RII_LIB=checked timeout 900 python tools/sanitize_driver.py tiny windows > gpurun_out/checked_drive_$T.log 2>&1; echo drive=$?
for f in checked_pytest_gpu checked_pytest_m8nth384 checked_drive; do tail -n 2 gpurun_out/${f}_$T.log; done
