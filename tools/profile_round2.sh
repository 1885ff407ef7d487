# Round-2 final profiling of the headline step (configs[1]): plain run, launch list with DRAM
# bytes (host-driven PCG loop so ncu attributes the kernels to the timed NVTX range), full
# captures of the four fine-level kernels with per-line source stalls.
R=${1:-r02f}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain.log; exit 1; }
tail -1 gpurun_out/plain.log | head -c 200; echo
NV='--nvtx --nvtx-include rbws_timed/'
RBWS_GRAPH=0 timeout 1200 ncu $NV --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo list=$?
CMD1="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 1200 ncu -f $NV --kernel-name-base demangled --set full --clock-control none --import-source on -k 'regex:(cgp_kernel|fine_kernel<\(int\)(5|6), \(int\)64)' -c 3 -o /tmp/${R}_fine $CMD1 > gpurun_out/ncu_fine.log 2>&1; echo fine=$?
ncu -i /tmp/${R}_fine.ncu-rep --page raw --csv > gpurun_out/${R}_fine_raw.csv 2>/dev/null
ncu -i /tmp/${R}_fine.ncu-rep --page source --csv > gpurun_out/${R}_fine_source.csv 2>/dev/null
python tools/ncu_source_summary.py gpurun_out/${R}_fine_source.csv 256047000 12 > gpurun_out/${R}_fine_summary.txt
python tools/launch_summary.py gpurun_out/${R}_launches.csv gpurun_out/${R}_launches.md gpurun_out/${R}_traffic.json > /dev/null
ls -la gpurun_out | tail -8
