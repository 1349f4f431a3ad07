# configs[4] IVF L = 64 (one 1,024-query call): launch list, then ncu --set full of the
# integer list-item kernel (last phase).
T=${TAG:-r02c}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/scale_ivf_launches_$T.csv python tools/scale_ab.py --profile > gpurun_out/scale_ivf_launches_$T.log 2>&1; echo launches=$?
timeout 1800 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.8, .int.8, .bool.1" --launch-skip 1 -c 1 -o gpurun_out/scale_ivf_$T python tools/scale_ab.py --profile > gpurun_out/ncu_scale_ivf_$T.log 2>&1; echo full=$?
ncu -i gpurun_out/scale_ivf_$T.ncu-rep --page raw --csv > gpurun_out/scale_ivf_${T}_raw.csv
ncu -i gpurun_out/scale_ivf_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/scale_ivf_${T}_src.csv
python tools/ncu_lines.py gpurun_out/scale_ivf_${T}_src.csv 40 > gpurun_out/scale_ivf_${T}_lines.txt
rm -f gpurun_out/scale_ivf_$T.ncu-rep gpurun_out/scale_ivf_${T}_src.csv
# the M = 8 linear scan (1,024 queries x 1e9 codes, one launch of the 16-query u6 kernel)
timeout 2400 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.8, .int.16, .bool.0" -c 1 -o gpurun_out/scale_lin_$T python tools/scale_ab.py --profile-linear > gpurun_out/ncu_scale_lin_$T.log 2>&1; echo lin=$?
ncu -i gpurun_out/scale_lin_$T.ncu-rep --page raw --csv > gpurun_out/scale_lin_${T}_raw.csv
ncu -i gpurun_out/scale_lin_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/scale_lin_${T}_src.csv
python tools/ncu_lines.py gpurun_out/scale_lin_${T}_src.csv 40 > gpurun_out/scale_lin_${T}_lines.txt
rm -f gpurun_out/scale_lin_$T.ncu-rep gpurun_out/scale_lin_${T}_src.csv
