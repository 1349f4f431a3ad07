# ncu --set full of the large-M chunked u6 kernel (GIST-like, M = 240, 10k queries, 1M codes).
T=${TAG:-0}
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_large_u6_kernel" --launch-skip ${SKIP:-1} -c 1 -o gpurun_out/large$T python tools/prof_query.py --workload gist1m --path linear > gpurun_out/ncu_large$T.log 2>&1; echo full=$?
ncu -i gpurun_out/large$T.ncu-rep --page raw --csv > gpurun_out/large${T}_raw.csv
ncu -i gpurun_out/large$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/large${T}_src.csv
python tools/ncu_lines.py gpurun_out/large${T}_src.csv 40 > gpurun_out/large${T}_lines.txt
rm -f gpurun_out/large$T.ncu-rep gpurun_out/large${T}_src.csv
