# Checked build over the GPU suite and the sanitizer drive (after the list-mode n_codes fix);
# bench line with the re-tied traffic; coarse top-P ROT_MINK A/B (sift1m M = 16, M = 64).
set -x
T=${TAG:-r02h}
RII_LIB=checked timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest_gpu_$T.log 2>&1; echo checked_gpu=$?
tail -3 gpurun_out/checked_pytest_gpu_$T.log
RII_LIB=checked timeout 900 python tools/sanitize_driver.py all > gpurun_out/checked_drive_$T.log 2>&1; echo checked_drive=$?
tail -5 gpurun_out/checked_drive_$T.log
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 9 --cases "ivf/1/0,ivf/4/0,ivf/16/0" "" "RII_COARSE_ROT_MINK=1" > gpurun_out/rotmink_sift_$T.jsonl 2>&1; echo ab=$?
timeout 900 python tools/ab_env.py --workload sift1m_m64 --reps 9 --cases "ivf/1/0,ivf/5/0" "" "RII_COARSE_ROT_MINK=1" > gpurun_out/rotmink_m64_$T.jsonl 2>&1; echo ab64=$?
