# Checked build (librii_b200_checked.so, RII_BOUNDS_CHECK: device-side bound asserts +
# a device sync after every launch) over the whole GPU suite and the sanitizer drive --
# the stand-in for compute-sanitizer, which this pool does not run; then the normal
# build: GPU suite, bench, launch list and ncu --set full of the headline (traffic
# re-tied to the sources' hash).
set -x
T=${TAG:-r02g}
RII_LIB=checked timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest_gpu_$T.log 2>&1; echo checked_gpu=$?
tail -3 gpurun_out/checked_pytest_gpu_$T.log
RII_LIB=checked timeout 900 python tools/sanitize_driver.py all > gpurun_out/checked_drive_$T.log 2>&1; echo checked_drive=$?
tail -5 gpurun_out/checked_drive_$T.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo gpu=$?
tail -2 gpurun_out/pytest_gpu_$T.log
timeout 500 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/ncu_l_$T.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k "regex:scan_fast_kernel<.int.32, .int.16, .bool.0" -c 1 -o gpurun_out/scan_$T python bench.py --no-extra --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_full_$T.log 2>&1; echo full=$?
ncu -i gpurun_out/scan_$T.ncu-rep --page raw --csv > gpurun_out/scan_${T}_raw.csv
ncu -i gpurun_out/scan_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/scan_${T}_src.csv
python tools/ncu_lines.py gpurun_out/scan_${T}_src.csv 40 > gpurun_out/scan_${T}_lines.txt
python tools/traffic_json.py gpurun_out/scan_${T}_raw.csv u6 "ncu --set full --clock-control none --profile-from-start off, profiles/${T}_scan_u6b16_raw.csv (bench.py --no-extra --no-cpu --steps 1 --warmup 3)" > gpurun_out/traffic_$T.json; echo traffic=$?
rm -f gpurun_out/scan_$T.ncu-rep gpurun_out/scan_${T}_src.csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?
