set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "u16_tables" tests/test_gpu_windows.py -x -q > gpurun_out/m5_tests.log 2>&1; echo tests=$?
timeout 900 python tools/ab_env.py --workload sift1m_m64 --path linear --reps 5 "" "RII_M64_NTH=384" "RII_M64_SPLIT=0" > gpurun_out/m5_m64.jsonl 2> gpurun_out/m5_m64.err; echo m64=$?
timeout 1500 python tools/ab_env.py --workload deep100m_m8 --reps 5 --cases "linear/64/1000000,ivf/64/0,ivf/64/1000000,linear/1/0" "" "RII_COARSE_TOPP=0" "RII_Q16_CFG=0" > gpurun_out/m5_m8.jsonl 2> gpurun_out/m5_m8.err; echo m8=$?
