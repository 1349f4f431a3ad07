set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/m8_gpu.log 2>&1; echo gpu=$?
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "ivf/64/0,ivf/16/0,ivf/1/0" "" > gpurun_out/m8_deep.jsonl 2>&1; echo ab=$?
timeout 2400 python tools/scale_ab.py "" "RII_LIST_PACKED_MIN=1000000000" "RII_LIST_BOUND=1" "RII_LIST_PHASES=1,2,4,8" > gpurun_out/m8_scale.jsonl 2> gpurun_out/m8_scale.err; echo scale=$?
TAG=r02c bash tools/ncu_scale_ivf.sh
