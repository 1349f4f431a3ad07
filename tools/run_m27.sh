# A/B: 512 threads against 384 for the M = 16, 16-query u6 linear kernel (RII_M16_NTH); the M = 8
# default (512) checked against its 384 variant by the extended u16/u6 test.
set -x
T=${TAG:-r02q}
RII_M16_NTH=512 timeout 900 python -m pytest tests/test_gpu_windows.py tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_masked.py -m gpu -q > gpurun_out/pytest_m16nth_$T.log 2>&1; echo par=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 7 --cases "linear/1/0,linear/1/0/1024,linear/1/100000" "" "RII_M16_NTH=512" "" "RII_M16_NTH=512" > gpurun_out/ab_m16nth_sift1m_$T.jsonl 2>&1; echo ab=$?
tail -2 gpurun_out/pytest_m16nth_$T.log; cat gpurun_out/ab_m16nth_sift1m_$T.jsonl | tail -20
