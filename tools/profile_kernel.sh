# ncu --set full (with per-line source stalls) of the first launches of one kernel in the
# headline step.   usage: bash tools/profile_kernel.sh <tag> <kernel regex> [count]
R=${1:-k}
K=${2:-coarse_tail}
C=${3:-1}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
NV='--nvtx --nvtx-include rbws_timed/'
timeout 1200 ncu -f $NV --kernel-name-base demangled --set full --clock-control none --import-source on -k "regex:$K" -c $C -o /tmp/${R} $CMD > gpurun_out/ncu_${R}.log 2>&1; echo ncu=$?
ncu -i /tmp/${R}.ncu-rep --page raw --csv > gpurun_out/${R}_raw.csv 2>/dev/null
ncu -i /tmp/${R}.ncu-rep --page source --csv > gpurun_out/${R}_source.csv 2>/dev/null
python tools/ncu_source_summary.py gpurun_out/${R}_source.csv ${4:-1} 25 > gpurun_out/${R}_summary.txt
