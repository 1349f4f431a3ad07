# Round-1 measurement pass: bench (ours + oracle arm), per-config table, launch list,
# one ncu --set full capture of the linear scan kernel (exported to CSV).
set -x
nvidia-smi -L
T=${TAG:-13}
timeout 400 python bench.py > gpurun_out/bench$T.json 2> gpurun_out/bench$T.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench${T}_ref.json 2>gpurun_out/bench${T}_ref.err; echo ref=$?
timeout 900 python tools/configs.py > gpurun_out/configs$T.jsonl 2> gpurun_out/configs$T.err; echo configs=$?
timeout 900 python tools/configs.py --only deep10m >> gpurun_out/configs$T.jsonl 2>> gpurun_out/configs$T.err; echo configs_deep=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches$T.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_l$T.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.16, .bool.0" -c 1 -o gpurun_out/scan$T python bench.py --no-extra --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_full$T.log 2>&1; echo full=$?
ncu -i gpurun_out/scan$T.ncu-rep --page raw --csv > gpurun_out/scan${T}_raw.csv
ncu -i gpurun_out/scan$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/scan${T}_src.csv
python tools/ncu_lines.py gpurun_out/scan${T}_src.csv 40 > gpurun_out/scan${T}_lines.txt
rm -f gpurun_out/scan$T.ncu-rep gpurun_out/scan${T}_src.csv
timeout 900 python tools/configs.py --only paper_t2 > gpurun_out/configs${T}_t2.jsonl 2> gpurun_out/configs${T}_t2.err; echo t2=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke$T.log 2>&1; echo smoke=$?
