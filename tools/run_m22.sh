# configs[4] (1e9 codes, M = 8) rows at HEAD, then the GPU suite at HEAD.
set -x
T=${TAG:-r02l}
timeout 1500 python tools/configs.py --only scale1b --reps 2 > gpurun_out/scale1b_$T.jsonl 2> gpurun_out/scale1b_$T.err; echo scale=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
tail -1 gpurun_out/pytest_gpu_$T.log
