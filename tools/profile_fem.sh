# Profiling recipe for the assembled-problem path (bench.py --problem example-1): plain run,
# launch list, one full capture of the batch-shared finest-level kernel and of the per-instance
# stored kernel (coarse levels).   usage: bash tools/profile_fem.sh r01f
R=${1:-r01f}
mkdir -p gpurun_out
CMD="python bench.py --problem example-1 --fem-n 64 --batch 256 --steps 1 --warmup 3 --no-cpu"
$CMD > gpurun_out/${R}_plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/${R}_plain.log; exit 1; }
tail -1 gpurun_out/${R}_plain.log | head -c 300; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_list.log 2>&1; echo list=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"stored_shared_kernel<2" -s 20 -c 2 -o /tmp/${R}_shared $CMD > gpurun_out/${R}_ncu_shared.log 2>&1; echo shared=$?
timeout 900 ncu -f --set full --clock-control none -k regex:"coarse_stored_kernel<2" -s 20 -c 2 -o /tmp/${R}_percoef $CMD > gpurun_out/${R}_ncu_percoef.log 2>&1; echo percoef=$?
for r in ${R}_shared ${R}_percoef; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
ncu -i /tmp/${R}_shared.ncu-rep --page source --csv > gpurun_out/${R}_shared_source.csv 2>/dev/null
ls -la gpurun_out/ | tail -12
