set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_masked.py tests/test_gpu_fullsize.py -x -q > gpurun_out/m14_gpu.log 2>&1; echo gpu=$?
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "ivf/1/0,ivf/64/0,ivf/64/1000000" "" "RII_COARSE_TOPP=0" > gpurun_out/m14_deep.jsonl 2>&1; echo ab=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 5 --cases "ivf/1/0,ivf/64/0,ivf/64/100000" "" > gpurun_out/m14_sift.jsonl 2>&1; echo ab=$?
