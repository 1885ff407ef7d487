mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu"
NV='--nvtx --nvtx-include rbws_timed/'
timeout 900 ncu $NV --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_slab4_launches.csv $CMD > gpurun_out/ncu_slab.log 2>&1; echo list=$?
tail -3 gpurun_out/ncu_slab.log
