# Profiling recipe (round R): plain run, launch list of the timed step, full captures of
# the fine-level kernels and the coarse/transfer kernels.  Reports stay in /tmp on the
# box; CSV exports come back in gpurun_out/.   usage: bash tools/profile_round.sh r01
R=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain.log; exit 1; }
tail -1 gpurun_out/plain.log | head -c 300; echo
NV='--nvtx --nvtx-include rbws_timed/'
timeout 900 ncu $NV --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo list=$?
timeout 900 ncu -f $NV --set full --clock-control none --import-source on -k regex:fine_kernel -c 12 -o /tmp/${R}_fine $CMD > gpurun_out/ncu_fine.log 2>&1; echo fine=$?
timeout 900 ncu -f $NV --set full --clock-control none -k regex:"coarse_kron|restrict|prolong" -c 10 -o /tmp/${R}_other $CMD > gpurun_out/ncu_other.log 2>&1; echo other=$?
for r in ${R}_fine ${R}_other; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
ncu -i /tmp/${R}_fine.ncu-rep --page source --csv > gpurun_out/${R}_fine_source.csv 2>/dev/null
ls -la gpurun_out/ | tail -12
