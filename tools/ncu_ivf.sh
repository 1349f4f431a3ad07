# ncu --set full of the list-major u6 item kernel (phase B) on deep10m IVF L=64.
T=${TAG:-0}
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.8, .bool.1, .int.(384|192)" --launch-skip 1 -c 1 -o gpurun_out/ivf$T python tools/prof_query.py --workload deep10m --path ivf --L 64 > gpurun_out/ncu_ivf$T.log 2>&1; echo full=$?
ncu -i gpurun_out/ivf$T.ncu-rep --page raw --csv > gpurun_out/ivf${T}_raw.csv
ncu -i gpurun_out/ivf$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ivf${T}_src.csv
python tools/ncu_lines.py gpurun_out/ivf${T}_src.csv 50 > gpurun_out/ivf${T}_lines.txt
ncu -i gpurun_out/ivf$T.ncu-rep --page details --csv > gpurun_out/ivf${T}_details.csv
rm -f gpurun_out/ivf$T.ncu-rep gpurun_out/ivf${T}_src.csv
