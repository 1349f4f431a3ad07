# A/B: 512 threads (16 warps per SM) against 384 for the M = 8, 16-query u6 linear kernel
# (RII_M8_NTH), parity of the variant first.
set -x
T=${TAG:-r02o}
RII_M8_NTH=512 timeout 900 python -m pytest tests/test_gpu_windows.py tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_masked.py -m gpu -q > gpurun_out/pytest_m8nth_$T.log 2>&1; echo par=$?
timeout 900 python tools/ab_env.py --workload deep10m_m8 --reps 5 --cases "linear/1/0,linear/1/0/1024,linear/1/1000000" "" "RII_M8_NTH=512" > gpurun_out/ab_m8nth_deep10m_$T.jsonl 2>&1; echo ab=$?
timeout 1200 python tools/ab_env.py --workload deep100m_m8 --reps 3 --cases "linear/1/0" "" "RII_M8_NTH=512" > gpurun_out/ab_m8nth_deep100m_$T.jsonl 2>&1; echo ab2=$?
tail -2 gpurun_out/pytest_m8nth_$T.log; cat gpurun_out/ab_m8nth_deep10m_$T.jsonl gpurun_out/ab_m8nth_deep100m_$T.jsonl | tail -20
