# A/B alternative builds of the library on configs[1]: bash tools/ab_libs.sh "" _v2 _v3
for v in "$@"; do
  RBWS_LIB=$PWD/paper_2311_13862_b200/_rbws_b200$v.so RBWS_PROF_DUMP=1 timeout 300 python bench.py --no-cpu 2>gpurun_out/pd$v.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lib$v', d['value'], d['e2e']['value'])"
  python - "$v" <<'PY'
import collections, sys
v = sys.argv[1]
rows=[l.split() for l in open(f'gpurun_out/pd{v}.txt') if l.startswith('PROF')]
rows=[(int(a),int(b),float(c)) for _,a,b,c in rows]
names={0:'papply',1:'cg',2:'pre',3:'restrict',4:'prolong',5:'post',6:'xpby',7:'coarse',8:'scal'}
full=collections.defaultdict(list)
for c,a,ms in rows:
    if a==1024: full[names[c]].append(ms)
print('   ', {k:round(sum(x)/len(x),3) for k,x in full.items()})
PY
done
