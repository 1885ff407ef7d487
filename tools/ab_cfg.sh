# A/B alternative builds of the library on another config: bash tools/ab_cfg.sh 2 "" _v2
C=$1; shift
for v in "$@"; do
  RBWS_LIB=$PWD/paper_2311_13862_b200/_rbws_b200$v.so timeout 900 python bench.py --config $C --steps 2 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('lib$v', d['value'], {k:v.get('ms_per_launch') for k,v in d['kernels'].items()})"
done
