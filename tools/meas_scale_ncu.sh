# ncu --set full of the M = 8 linear scan kernel on configs[4] (1e9 codes, 1024 queries):
# which pipe bounds it and how often the 8 GB of codes are re-streamed from DRAM.
T=${TAG:-r02}
RII_PROFILE_LINEAR=1 timeout 2400 ncu --set full --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.8, .int.8" -c 1 -o gpurun_out/scale1b_$T python tools/configs.py --only scale1b --reps 1 > gpurun_out/scale1b_ncu_$T.log 2>&1; echo ncu=$?
ncu -i gpurun_out/scale1b_$T.ncu-rep --page raw --csv > gpurun_out/scale1b_${T}_raw.csv
rm -f gpurun_out/scale1b_$T.ncu-rep
