# Round-2 final measurement pass (TAG=r02c): GPU tests, bench + oracle arm, launch list, ncu of the
# headline and IVF item kernels, per-config rows, Table-2 shapes, configs[4] rows, smoke, IVF A/B.
set -x
T=${TAG:-r02c}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
TAG=$T bash tools/meas_r2.sh
TAG=$T bash tools/meas_scale.sh
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "ivf/64/0,ivf/16/0" "" "RII_LIST_BOUND=1" > gpurun_out/ab_listbound_$T.jsonl 2>&1; echo ab=$?
RII_TRACE=1 timeout 600 python tools/prof_query.py --path ivf --L 64 --reps 1 > gpurun_out/trace_ivf64_$T.log 2>&1; echo trace=$?
