# deep10m IVF L = 64: ncu --set full of the first integer list-item launch (phase 1, ranks [1, 4))
# and of the rank-0 fp32 items (phase 0), for the per-phase cost study.
T=${TAG:-r02d}
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.8, .bool.1, .int.(384|192)" -c 1 -o gpurun_out/ivfp1_$T python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_ivfp1_$T.log 2>&1; echo p1=$?
ncu -i gpurun_out/ivfp1_$T.ncu-rep --page raw --csv > gpurun_out/ivfp1_${T}_raw.csv
ncu -i gpurun_out/ivfp1_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ivfp1_${T}_src.csv
python tools/ncu_lines.py gpurun_out/ivfp1_${T}_src.csv 40 > gpurun_out/ivfp1_${T}_lines.txt
rm -f gpurun_out/ivfp1_$T.ncu-rep gpurun_out/ivfp1_${T}_src.csv
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.6, .bool.1" -c 1 -o gpurun_out/ivfp0_$T python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_ivfp0_$T.log 2>&1; echo p0=$?
ncu -i gpurun_out/ivfp0_$T.ncu-rep --page raw --csv > gpurun_out/ivfp0_${T}_raw.csv
ncu -i gpurun_out/ivfp0_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ivfp0_${T}_src.csv
python tools/ncu_lines.py gpurun_out/ivfp0_${T}_src.csv 40 > gpurun_out/ivfp0_${T}_lines.txt
rm -f gpurun_out/ivfp0_$T.ncu-rep gpurun_out/ivfp0_${T}_src.csv
RII_DBG_MASK=4 timeout 600 python tools/prof_query.py --workload deep10m --path ivf --L 64 --counters > gpurun_out/counters_ivf64_$T.log 2>&1; echo counters=$?
