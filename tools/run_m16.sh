# Re-entry validation at HEAD (after the RII_COARSE_ROT_MINK change): full GPU suite,
# smoke, bench line, the m15 coarse A/B.
set -x
T=${TAG:-r02f}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 600 python tools/ab_env.py --workload sift1m --reps 5 --cases "ivf/1/0,ivf/4/0,ivf/64/0" "" "RII_COARSE_ROT_MINK=1" > gpurun_out/m16_sift.jsonl 2>&1; echo ab=$?
