# configs[4] (1e9 codes, M = 8) on one B200 at HEAD: build rows, IVF / subset / linear rows,
# then an ncu --set full capture of the M = 8 linear scan kernel (one launch).
T=${TAG:-r02}
timeout 1500 python tools/configs.py --only scale1b --reps 2 > gpurun_out/scale1b_$T.jsonl 2> gpurun_out/scale1b_$T.err; echo scale=$?
