# A/B: 512 against 384 threads for short M = 8 scans (configs[4]'s subset row shape: 1,024 queries
# per call over a gathered 1e6-code subset; also 1e5 / 1e4 ids and small query batches).
set -x
T=${TAG:-r02r}
timeout 900 python tools/ab_env.py --workload deep10m_m8 --reps 9 --cases "linear/1/1000000/1024,linear/1/100000/1024,linear/1/100000,linear/1/10000,linear/1/1000000/128,linear/1/0/128" "" "RII_M8_NTH=384" "" "RII_M8_NTH=384" > gpurun_out/ab_m8nth_short_$T.jsonl 2>&1; echo ab=$?
