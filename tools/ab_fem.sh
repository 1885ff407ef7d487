# A/B of stored_shared_kernel variants on the box (rebuilds with RBWS_EXTRA_DEFS per variant)
mkdir -p gpurun_out
B="python bench.py --problem example-1 --fem-n 64 --batch 256 --steps 3 --warmup 3 --no-cpu"
for v in "RBWS_SHARED_UNROLL=13" "RBWS_SHARED_UNROLL=2" "RBWS_SHARED_UNROLL=4" "RBWS_SHARED_UNROLL=1" "RBWS_SHARED_UNROLL=13 RBWS_SHARED_MINB=1"; do
  RBWS_EXTRA_DEFS="$v" python build.py --force > gpurun_out/ab_build.log 2>&1 || { echo build failed $v; continue; }
  $B > gpurun_out/ab.log 2>&1
  echo "$v" $(grep -o "\"value\": [0-9.]*" gpurun_out/ab.log | head -1) $(grep -o "\"ms_per_launch\": [0-9.]*" gpurun_out/ab.log)
done
