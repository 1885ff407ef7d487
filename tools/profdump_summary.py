"""Per-class full-batch kernel times from RBWS_PROF_DUMP=1 bench runs (stderr dumps)."""
import collections
import sys

names = {0: 'papply', 1: 'cg', 2: 'pre', 3: 'restrict', 4: 'prolong', 5: 'post', 6: 'xpby',
         7: 'coarse', 8: 'scal'}
for path in sys.argv[1:]:
    rows = [l.split() for l in open(path) if l.startswith('PROF')]
    rows = [(int(a), int(b), float(c)) for _, a, b, c in rows]
    top = max(a for _, a, _ in rows)
    full = collections.defaultdict(list)
    for c, a, ms in rows:
        if a == top:
            full[names.get(c, c)].append(ms)
    print(path, top, {k: round(sum(v) / len(v), 3) for k, v in full.items()})
