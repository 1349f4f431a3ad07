set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/m3_gpu.log 2>&1; echo gpu=$?
for L in 1 4 16 64; do
 timeout 600 python tools/prof_query.py --path ivf --L $L --reps 5 >> gpurun_out/m3_ab.log 2>&1
 RII_COARSE_TOPP=0 timeout 600 python tools/prof_query.py --path ivf --L $L --reps 5 >> gpurun_out/m3_ab.log 2>&1
done
RII_TRACE=1 timeout 600 python tools/prof_query.py --path ivf --L 64 --subset 0.1 --reps 2 > gpurun_out/m3_trace.log 2>&1; echo trace=$?
timeout 900 python tools/configs.py --only sift1m,deep10m > gpurun_out/m3_configs.jsonl 2> gpurun_out/m3_configs.err; echo configs=$?
