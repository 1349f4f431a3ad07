# Sample size of the linear bound pass (RII_Q16_SAMPLE) on the headline workload.
set -x
T=${TAG:-r02m}
timeout 900 python tools/ab_env.py --workload deep10m --reps 5 --cases "linear/1/0" "" "RII_Q16_SAMPLE=16384" "RII_Q16_SAMPLE=8192" "RII_Q16_SAMPLE=65536" > gpurun_out/q16sample_deep_$T.jsonl 2>&1; echo ab=$?
timeout 600 python tools/ab_env.py --workload sift1m --reps 5 --cases "linear/1/0" "" "RII_Q16_SAMPLE=16384" "RII_Q16_SAMPLE=8192" > gpurun_out/q16sample_sift_$T.jsonl 2>&1; echo ab2=$?
