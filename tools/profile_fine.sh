# ncu --set full of the headline step's PREX / POSTP / PAPPLY kernels with per-line source
# stalls.   usage: bash tools/profile_fine.sh r02a
R=${1:-r02a}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain.log; exit 1; }
NV='--nvtx --nvtx-include rbws_timed/'
timeout 1200 ncu -f $NV --kernel-name-base demangled --set full --clock-control none --import-source on -k 'regex:fine_kernel<\(int\)(7|6|5), \(int\)64' -c 3 -o /tmp/${R}_fine $CMD > gpurun_out/ncu_fine.log 2>&1; echo fine=$?
ncu -i /tmp/${R}_fine.ncu-rep --page raw --csv > gpurun_out/${R}_fine_raw.csv 2>/dev/null
ncu -i /tmp/${R}_fine.ncu-rep --page details --csv > gpurun_out/${R}_fine_details.csv 2>/dev/null
ncu -i /tmp/${R}_fine.ncu-rep --page source --csv > gpurun_out/${R}_fine_source.csv 2>/dev/null
ls -la gpurun_out/ | tail -5
