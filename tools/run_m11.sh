set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/m11_gpu.log 2>&1; echo gpu=$?
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "ivf/1/0,ivf/4/0,ivf/64/0,ivf/64/1000000" "" "RII_COARSE_TOPP=0" > gpurun_out/m11_deep.jsonl 2>&1; echo ab=$?
timeout 900 python tools/ab_env.py --workload sift1m --reps 5 --cases "ivf/1/0,ivf/64/0" "" "RII_COARSE_TOPP=0" > gpurun_out/m11_sift.jsonl 2>&1; echo ab=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:coarse_topp_kernel" -c 1 -o gpurun_out/coarse_r02e python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_coarse_r02e.log 2>&1; echo coarse=$?
ncu -i gpurun_out/coarse_r02e.ncu-rep --page raw --csv > gpurun_out/coarse_r02e_raw.csv; rm -f gpurun_out/coarse_r02e.ncu-rep
TAG=r02d bash tools/ncu_phase1.sh
