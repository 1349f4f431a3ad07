# Round-2 measurement pass at HEAD: bench (ours + oracle arm), launch list, ncu --set full of the
# headline kernel (-> profiles/scan_traffic.json, tied to the kernel sources' hash), ncu of the IVF
# list-major u6 items, per-config rows, paper Table 2 shapes, smoke.
set -x
T=${TAG:-r02}
nvidia-smi -L
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/ncu_l_$T.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.16, .bool.0" -c 1 -o gpurun_out/scan_$T python bench.py --no-extra --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_full_$T.log 2>&1; echo full=$?
ncu -i gpurun_out/scan_$T.ncu-rep --page raw --csv > gpurun_out/scan_${T}_raw.csv
ncu -i gpurun_out/scan_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/scan_${T}_src.csv
python tools/ncu_lines.py gpurun_out/scan_${T}_src.csv 40 > gpurun_out/scan_${T}_lines.txt
python tools/traffic_json.py gpurun_out/scan_${T}_raw.csv u6 "ncu --set full --clock-control none --profile-from-start off, profiles/${T}_scan_u6b16_raw.csv (bench.py --no-extra --no-cpu --steps 1 --warmup 3)" > gpurun_out/traffic_$T.json; echo traffic=$?
rm -f gpurun_out/scan_$T.ncu-rep gpurun_out/scan_${T}_src.csv
TAG=$T bash tools/ncu_ivf.sh
timeout 900 python tools/configs.py --only tiny,sift1m,growth > gpurun_out/configs_$T.jsonl 2> gpurun_out/configs_$T.err; echo configs=$?
timeout 900 python tools/configs.py --only deep10m >> gpurun_out/configs_$T.jsonl 2>> gpurun_out/configs_$T.err; echo configs_deep=$?
timeout 900 python tools/configs.py --only paper_t2 > gpurun_out/configs_${T}_t2.jsonl 2> gpurun_out/configs_${T}_t2.err; echo t2=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
