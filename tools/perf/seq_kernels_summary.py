import collections, csv, sys
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0].isdigit()]
    c = collections.defaultdict(list)
    for r in rows:
        c[r[4].split('(')[0].replace('void ', '').replace('mdhp::', '')].append(float(r[-1]))
    it = [k for k in c if any(s in k for s in ('local', 'scan', 'eval', 'reduce', 'finish'))]
    tot = sum(sorted(c[k])[len(c[k]) // 2] for k in it)
    print(f, ' '.join(f"{k.split('<')[0][6:]}={sorted(c[k])[len(c[k]) // 2] / 1e3:.1f}" for k in it), f"iter={tot / 1e3:.1f}us")
