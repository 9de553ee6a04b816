"""Per-chunk table of a batch-pipeline timeline (SA_DEBUG_TIMELINE=1 stderr
lines): event times after each chunk's H2D, seed, solo, resolve, warp,
prune, overflow pass and D2H.  python scripts/timeline_table.py LOG"""
import sys, collections
lines = [l.split() for l in open(sys.argv[1]) if l.startswith('[tl]')]
# split batches: a new batch starts when chunk 0 'C' appears
batches, cur = [], []
for _, c, t, v in lines:
    if c == '0' and t == 'C' and cur: batches.append(cur); cur = []
    cur.append((int(c), t, float(v)))
batches.append(cur)
b = batches[-1]
tab = collections.defaultdict(dict)
for c, t, v in b: tab[c][t] = v
print('chunk   C(h2d)  S(seed)  o(solo) r(res)  w(warp)  p(prune) V(ovf)  D(d2h)')
for c in sorted(tab):
    d = tab[c]
    print(f"{c:4d} " + " ".join(f"{d.get(t, float('nan')):8.2f}" for t in "CSorwpVD"))
