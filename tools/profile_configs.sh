# ncu launch lists (time + DRAM bytes per launch) of the timed step of configs 2 and 3,
# each after the same command ran clean without ncu.  usage: bash tools/profile_configs.sh r01e
R=${1:-r01e}
mkdir -p gpurun_out
NV='--nvtx --nvtx-include rbws_timed/'
for c in 2 3; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu"
  $CMD > gpurun_out/plain$c.log 2>&1 || { echo "config $c failed"; tail -3 gpurun_out/plain$c.log; continue; }
  timeout 1200 ncu $NV --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/${R}_cfg${c}_launches.csv $CMD > gpurun_out/ncu_cfg$c.log 2>&1; echo "cfg$c ncu=$?"
done
