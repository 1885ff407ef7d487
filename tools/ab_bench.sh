# quick A/B of the configs[1] step: gpu tests, then per-class full-batch kernel times
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
RBWS_PROF_DUMP=1 timeout 300 python bench.py --no-cpu 2>gpurun_out/profdump.txt | tail -1 | cut -c1-200
python - <<'PY'
import collections
rows=[l.split() for l in open('gpurun_out/profdump.txt') if l.startswith('PROF')]
rows=[(int(a),int(b),float(c)) for _,a,b,c in rows]
names={0:'papply',1:'cg',2:'pre',3:'restrict',4:'prolong',5:'post',6:'xpby',7:'coarse',8:'scal'}
full=collections.defaultdict(list)
for c,a,ms in rows:
    if a==1024: full[names[c]].append(ms)
print({k:round(sum(v)/len(v),3) for k,v in full.items()})
PY
