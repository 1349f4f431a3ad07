# Diagnosis (no source change): why 512 threads lose on few query batches over a long M = 8 scan --
# with / without the L2 prefetch, and with the chunk length fixed.
set -x
T=${TAG:-r02u}
timeout 900 python tools/ab_env.py --workload deep10m_m8 --reps 7 --cases "linear/1/0/128,linear/1/0/256" "RII_M8_NTH=384" "RII_M8_NTH=512" "RII_M8_NTH=384;RII_LIN_PF=0" "RII_M8_NTH=512;RII_LIN_PF=0" "RII_M8_NTH=384;RII_CHUNK_CODES=1000000" "RII_M8_NTH=512;RII_CHUNK_CODES=1000000" "RII_M8_NTH=384;RII_CHUNK_CODES=250000" "RII_M8_NTH=512;RII_CHUNK_CODES=250000" > gpurun_out/ab_m8nth_diag_$T.jsonl 2>&1; echo ab=$?
