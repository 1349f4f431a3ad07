# Rank-0 phase on the query-major traversal (RII_R0_QMAJOR): parity (new test + IVF suites),
# A/B on deep10m / sift1m IVF rows.
set -x
T=${TAG:-r02j}
timeout 1200 python -m pytest tests/test_gpu_masked.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_r0q_$T.log 2>&1; echo gpu=$?
tail -3 gpurun_out/pytest_r0q_$T.log
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "ivf/4/0,ivf/16/0,ivf/64/0" "" "RII_R0_QMAJOR=0" > gpurun_out/r0q_deep_$T.jsonl 2>&1; echo ab=$?
timeout 600 python tools/ab_env.py --workload sift1m --reps 7 --cases "ivf/16/0,ivf/64/0" "" "RII_R0_QMAJOR=0" > gpurun_out/r0q_sift_$T.jsonl 2>&1; echo ab2=$?
