set -x
TAG=r02c bash tools/ncu_scale_ivf.sh
timeout 2400 python tools/scale_ab.py "" "RII_LIST_PACKED_MIN=1000000000" "RII_LIST_BOUND=1" "RII_LIST_PHASES=1,2,4,8" > gpurun_out/m8_scale.jsonl 2> gpurun_out/m8_scale.err; echo scale=$?
