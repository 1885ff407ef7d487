# bench line of every BASELINE config (one B200) -> gpurun_out/cfg<C>.log
mkdir -p gpurun_out
for c in 0 1 2 3 4; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/cfg$c.log 2>&1
  echo "config $c rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/cfg$c.log | head -2 | tr '\n' ' ')"
done
