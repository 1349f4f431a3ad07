# IVF timing pass (deep10m / sift1m, several L and subsets) with the current build.
# usage: TAG=x bash tools/ivf_ab.sh   (writes gpurun_out/ivf_$TAG.log)
T=${TAG:-0}
O=gpurun_out/ivf_$T.log
: > $O
for L in 64 16 4 1; do timeout 300 python tools/prof_query.py --workload deep10m --path ivf --L $L --reps 5 >> $O 2>&1; done
timeout 300 python tools/prof_query.py --workload deep10m --path ivf --L 64 --subset 0.1 --reps 3 >> $O 2>&1
timeout 300 python tools/prof_query.py --workload deep10m --path ivf --L 64 --subset 0.01 --reps 3 >> $O 2>&1
timeout 300 python tools/prof_query.py --workload sift1m --path ivf --L 64 --reps 5 >> $O 2>&1
timeout 300 python tools/prof_query.py --workload sift1m --path ivf --L 16 --reps 5 >> $O 2>&1
timeout 300 python tools/prof_query.py --workload sift1m_m64 --path ivf --L 5 --reps 5 >> $O 2>&1
