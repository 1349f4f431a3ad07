set -x
timeout 2400 python tools/scale_ab.py "" "RII_COARSE_TOPP=0" "RII_Q16_CFG=0" "RII_LIST_U7=0" > gpurun_out/m7_scale.jsonl 2> gpurun_out/m7_scale.err; echo scale=$?
