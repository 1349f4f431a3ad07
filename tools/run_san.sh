# compute-sanitizer over every kernel family (tools/sanitize_driver.py), one tool per call:
#   TOOL=memcheck|racecheck|synccheck|initcheck bash tools/run_san.sh
set -x
TOOL=${TOOL:-memcheck}
for part in ${PARTS:-tiny windows ivf masked}; do
  timeout ${TMO:-900} compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_driver.py $part > gpurun_out/san_${TOOL}_$part.log 2>&1; echo $TOOL $part=$?
  tail -3 gpurun_out/san_${TOOL}_$part.log
done
