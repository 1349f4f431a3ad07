# Round-2 final measurement pass: GPU tests, bench + oracle arm, launch list, ncu of the headline
# and IVF item kernels, per-config rows, Table-2 shapes, configs[4] rows + ncu, smoke, traces.
set -x
T=${TAG:-r02d}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
TAG=$T bash tools/meas_r2.sh
TAG=$T bash tools/meas_scale.sh
TAG=$T bash tools/ncu_scale_ivf.sh
RII_TRACE=1 timeout 600 python tools/prof_query.py --path ivf --L 64 --reps 1 > gpurun_out/trace_ivf64_$T.log 2>&1; echo trace=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:coarse_topp_kernel" -c 1 -o gpurun_out/coarse_$T python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_coarse_$T.log 2>&1; echo coarse=$?
ncu -i gpurun_out/coarse_$T.ncu-rep --page raw --csv > gpurun_out/coarse_${T}_raw.csv; rm -f gpurun_out/coarse_$T.ncu-rep
timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.16, .bool.0" -c 1 -o gpurun_out/masked_$T python tools/prof_query.py --workload deep10m --path ivf --L 64 --subset 0.1 > gpurun_out/ncu_masked_$T.log 2>&1; echo masked=$?
ncu -i gpurun_out/masked_$T.ncu-rep --page raw --csv > gpurun_out/masked_${T}_raw.csv; rm -f gpurun_out/masked_$T.ncu-rep
