# Closing pass after the M = 8 thread-count gate (same steps as run_m26.sh, then the gate A/B).
# (-> profiles/scan_traffic.json tied to the sources' hash), launch list, both bench arms.
set -x
T=${TAG:-r02s}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.16, .bool.0" -c 1 -o gpurun_out/scan_$T python bench.py --no-extra --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_full_$T.log 2>&1; echo full=$?
ncu -i gpurun_out/scan_$T.ncu-rep --page raw --csv > gpurun_out/scan_${T}_raw.csv
ncu -i gpurun_out/scan_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/scan_${T}_src.csv
python tools/ncu_lines.py gpurun_out/scan_${T}_src.csv 40 > gpurun_out/scan_${T}_lines.txt
python tools/traffic_json.py gpurun_out/scan_${T}_raw.csv u6 "ncu --set full --clock-control none --profile-from-start off, profiles/${T}_scan_u6b16_raw.csv (bench.py --no-extra --no-cpu --steps 1 --warmup 3)" > gpurun_out/traffic_$T.json; echo traffic=$?
rm -f gpurun_out/scan_$T.ncu-rep gpurun_out/scan_${T}_src.csv
cp gpurun_out/traffic_$T.json profiles/scan_traffic.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/ncu_l_$T.log 2>&1; echo launches=$?
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 500 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo ref=$?
tail -2 gpurun_out/pytest_gpu_$T.log; cat gpurun_out/bench_$T.json | cut -c1-1500
# the M = 8 thread-count gate (m8_nth): default against either forced configuration
timeout 900 python tools/ab_env.py --workload deep10m_m8 --reps 7 --cases "linear/1/0/128,linear/1/0/256,linear/1/0/512,linear/1/0/1024,linear/1/0,linear/1/1000000/128" "" "RII_M8_NTH=384" "RII_M8_NTH=512" > gpurun_out/ab_m8nth_gate_$T.jsonl 2>&1; echo ab=$?
