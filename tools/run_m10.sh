set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/m10_gpu.log 2>&1; echo gpu=$?
RII_LIN_PF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -k "u16_tables or paths_match" tests/test_gpu_windows.py -x -q > gpurun_out/m10_tests_pf.log 2>&1; echo tests_pf=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 5 --cases "linear/1/0" "" "RII_LIN_PF=1" > gpurun_out/m10_sift.jsonl 2>&1; echo ab=$?
timeout 900 python tools/ab_env.py --workload deep10m_m8 --reps 3 --cases "linear/1/0,ivf/64/0" "" "RII_LIN_PF=1" > gpurun_out/m10_m8.jsonl 2>&1; echo ab=$?
timeout 2400 python tools/scale_ab.py "" "RII_LIN_PF=1" > gpurun_out/m10_scale.jsonl 2> gpurun_out/m10_scale.err; echo scale=$?
