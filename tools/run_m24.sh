# Re-entry validation at the round-2 head (fresh container, rebuilt library): GPU tests,
# smoke, both bench arms, launch list of the bench command.
set -x
T=${TAG:-r02n}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 500 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch_$T.log 2>&1; echo launches=$?
tail -3 gpurun_out/pytest_gpu_$T.log; cat gpurun_out/bench_$T.json
