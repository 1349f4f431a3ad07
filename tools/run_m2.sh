set -x
timeout 900 python -m pytest tests/test_gpu_masked.py -x -q > gpurun_out/m2_masked.log 2>&1; echo masked=$?
RII_TRACE=1 timeout 600 python tools/prof_query.py --path ivf --L 64 --subset 0.1 --reps 2 > gpurun_out/m2_trace.log 2>&1; echo trace=$?
RII_TRACE=1 timeout 600 python tools/prof_query.py --path linear --L 64 --subset 0.1 --reps 2 >> gpurun_out/m2_trace.log 2>&1; echo trace=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/m2_gpu.log 2>&1; echo gpu=$?
