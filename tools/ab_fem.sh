mkdir -p gpurun_out
B="python bench.py --problem example-1 --fem-n 64 --batch 256 --steps 3 --warmup 3 --no-cpu"
$B > gpurun_out/abA.log 2>&1; echo A $(grep -o "\"value\": [0-9.]*" gpurun_out/abA.log | head -1) $(grep -o "\"ms_per_launch\": [0-9.]*" gpurun_out/abA.log)
timeout 600 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stored_shared_kernel<2" -s 20 -c 1 -o /tmp/r01f_shared python bench.py --problem example-1 --fem-n 64 --batch 256 --steps 1 --warmup 3 --no-cpu > gpurun_out/r01f_ncu_shared.log 2>&1; echo ncu=$?
ncu -i /tmp/r01f_shared.ncu-rep --page raw --csv > gpurun_out/r01f_shared_raw.csv 2>/dev/null
ncu -i /tmp/r01f_shared.ncu-rep --page details --csv > gpurun_out/r01f_shared_details.csv 2>/dev/null
ncu -i /tmp/r01f_shared.ncu-rep --page source --csv > gpurun_out/r01f_shared_source.csv 2>/dev/null
RBWS_EXTRA_DEFS="RBWS_SHARED_MINB=3" python build.py --force > gpurun_out/buildB.log 2>&1; echo buildB=$?
$B > gpurun_out/abB.log 2>&1; echo B $(grep -o "\"value\": [0-9.]*" gpurun_out/abB.log | head -1) $(grep -o "\"ms_per_launch\": [0-9.]*" gpurun_out/abB.log)
