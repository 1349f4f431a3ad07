# Rank-0 query-major phase with lists split over warps (RII_R0_NSEG): A/B on deep10m.
set -x
T=${TAG:-r02k}
timeout 600 python -m pytest tests/test_gpu_masked.py -x -q -k rank0 > gpurun_out/pytest_r0q_$T.log 2>&1; echo gpu=$?
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "ivf/16/0,ivf/64/0" "RII_R0_QMAJOR=0" "RII_R0_NSEG=4" "RII_R0_NSEG=8" "RII_R0_NSEG=16" > gpurun_out/r0q_deep_$T.jsonl 2>&1; echo ab=$?
