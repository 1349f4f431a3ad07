set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_masked.py -x -q > gpurun_out/m1_masked.log 2>&1; echo masked=$?
timeout 900 python tools/configs.py --only sift1m,deep10m > gpurun_out/m1_configs.jsonl 2> gpurun_out/m1_configs.err; echo configs=$?
timeout 400 python bench.py --no-cpu > gpurun_out/m1_bench.json 2> gpurun_out/m1_bench.err; echo bench=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/m1_gpu.log 2>&1; echo gpu=$?
