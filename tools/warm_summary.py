import sys, collections
sys.path.insert(0, 'tools')
from ncu_summary import load
for f in sys.argv[1:]:
    r = load(f); n = len(r)
    # profile_target: cold invoke (no-overlap: swap + layer kernels + finish) then warm invokes
    k = [i for i, x in enumerate(r) if 'k_finish' in x[1]]
    warm = r[k[0] + 1:k[1] + 1] if len(k) > 1 else r
    fam = collections.defaultdict(list)
    for _, nm, ns in warm: fam[nm.split('(')[0][-24:]].append(ns / 1e3)
    print(f, 'warm kernels', len(warm), 'sum %.1f us' % sum(x[2] for x in warm) / 1 if False else '', 'sum us = %.1f' % (sum(x[2] for x in warm) / 1e3))
    for kk, v in sorted(fam.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {kk:26s} n={len(v):3d} sum={sum(v):8.1f} mean={sum(v)/len(v):6.2f} min={min(v):6.2f} max={max(v):6.2f}")
