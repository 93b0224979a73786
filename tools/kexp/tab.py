"""Tabulate a kexp log: add/contains Gkeys/s and contains registers per variant."""
import json
import sys

cur = None
rows = {}
for l in open(sys.argv[1]):
    if l.startswith('=='):
        cur = l.split()[1].replace('kexp_', '')
        continue
    try:
        r = json.loads(l)
    except ValueError:
        print(l.rstrip())
        continue
    rows.setdefault(r['cfg'], {})[cur] = (r['add'], r['contains'], r['regs_c'], r['out_hash'], r['filter_hash'])
vs = sorted({v for d in rows.values() for v in d})
print('cfg'.ljust(20), ' '.join(v.rjust(14) for v in vs))
for c, d in rows.items():
    print(c.ljust(20), ' '.join(('%.0f/%.0f r%d' % d[v][:3]).rjust(14) if v in d else '-'.rjust(14) for v in vs),
          '' if len({d[v][3:] for v in d}) == 1 else 'MISMATCH')
