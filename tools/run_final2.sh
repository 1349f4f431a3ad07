# Round-2 closing pass after the coarse-kernel changes (k_ivf.cu only; the linear scan and
# bench sources are those of r02d): GPU tests, per-config rows, Table-2 shapes, smoke, trace,
# ncu of the coarse top-P kernel, bench line.
set -x
T=${TAG:-r02e}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 900 python tools/configs.py --only tiny,sift1m,growth > gpurun_out/configs_$T.jsonl 2> gpurun_out/configs_$T.err; echo configs=$?
timeout 900 python tools/configs.py --only deep10m >> gpurun_out/configs_$T.jsonl 2>> gpurun_out/configs_$T.err; echo configs_deep=$?
timeout 900 python tools/configs.py --only paper_t2 > gpurun_out/configs_${T}_t2.jsonl 2> gpurun_out/configs_${T}_t2.err; echo t2=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
RII_TRACE=1 timeout 600 python tools/prof_query.py --path ivf --L 64 --reps 1 > gpurun_out/trace_ivf64_$T.log 2>&1; echo trace=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:coarse_topp_kernel" -c 1 -o gpurun_out/coarse_$T python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_coarse_$T.log 2>&1; echo coarse=$?
ncu -i gpurun_out/coarse_$T.ncu-rep --page raw --csv > gpurun_out/coarse_${T}_raw.csv; rm -f gpurun_out/coarse_$T.ncu-rep
