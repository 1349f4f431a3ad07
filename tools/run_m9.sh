set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/m9_gpu.log 2>&1; echo gpu=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 5 --cases "ivf/64/0,ivf/16/0" "" "RII_LIST_U=1" > gpurun_out/m9_sift.jsonl 2>&1; echo ab=$?
timeout 900 python tools/ab_env.py --workload deep10m_m8 --reps 5 --cases "ivf/64/0,ivf/16/0" "" "RII_LIST_U=1" > gpurun_out/m9_m8.jsonl 2>&1; echo ab=$?
timeout 2400 python tools/scale_ab.py "" "RII_LIST_U=1" "RII_LIST_PACKED_MIN=1000000000" > gpurun_out/m9_scale.jsonl 2> gpurun_out/m9_scale.err; echo scale=$?
