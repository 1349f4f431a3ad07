# After the coarse ROT_MINK default change: GPU suite (product and checked builds), drive,
# smoke, bench, per-config rows and Table-2 shapes.
set -x
T=${TAG:-r02i}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
tail -2 gpurun_out/pytest_gpu_$T.log
RII_LIB=checked timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest_gpu_$T.log 2>&1; echo checked_gpu=$?
tail -2 gpurun_out/checked_pytest_gpu_$T.log
RII_LIB=checked timeout 900 python tools/sanitize_driver.py all > gpurun_out/checked_drive_$T.log 2>&1; echo checked_drive=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 900 python tools/configs.py --only tiny,sift1m,growth > gpurun_out/configs_$T.jsonl 2> gpurun_out/configs_$T.err; echo configs=$?
timeout 900 python tools/configs.py --only deep10m >> gpurun_out/configs_$T.jsonl 2>> gpurun_out/configs_$T.err; echo configs_deep=$?
timeout 900 python tools/configs.py --only paper_t2 > gpurun_out/configs_${T}_t2.jsonl 2> gpurun_out/configs_${T}_t2.err; echo t2=$?
