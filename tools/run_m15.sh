set -x
timeout 1500 python -m pytest tests/test_gpu_masked.py tests/test_gpu_parity.py -x -q > gpurun_out/m15_gpu.log 2>&1; echo gpu=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 7 --cases "ivf/1/0,ivf/4/0,ivf/64/0" "" "RII_COARSE_ROT_MINK=1" > gpurun_out/m15_sift.jsonl 2>&1; echo ab=$?
timeout 900 python tools/ab_env.py --workload sift1m_m64 --reps 7 --cases "ivf/5/0" "" "RII_COARSE_ROT_MINK=1" > gpurun_out/m15_m64.jsonl 2>&1; echo ab=$?
