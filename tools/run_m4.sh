set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/m4_gpu.log 2>&1; echo gpu=$?
TAG=r02b bash tools/meas_r2.sh
TAG=r02b bash tools/meas_scale.sh
timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:coarse_topp_kernel" -c 1 -o gpurun_out/coarse_r02b python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_coarse_r02b.log 2>&1; echo coarse=$?
ncu -i gpurun_out/coarse_r02b.ncu-rep --page raw --csv > gpurun_out/coarse_r02b_raw.csv; rm -f gpurun_out/coarse_r02b.ncu-rep
timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.16, .bool.0" -c 1 -o gpurun_out/masked_r02b python tools/prof_query.py --workload deep10m --path ivf --L 64 --subset 0.1 > gpurun_out/ncu_masked_r02b.log 2>&1; echo masked=$?
ncu -i gpurun_out/masked_r02b.ncu-rep --page raw --csv > gpurun_out/masked_r02b_raw.csv; rm -f gpurun_out/masked_r02b.ncu-rep
