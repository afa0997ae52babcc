"""Summarise ncu source-page stall samples per role (producer/consumer) and reason."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
srcs = [r[1].strip() for r in data]
split = [i for i, s in enumerate(srcs) if 'USETMAXREG.DEALLOC' in s]
split = split[0] if split else len(data)
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
for name, lo, hi in [('producer', 0, split), ('consumer', split, len(data))]:
    tot = {}
    for r in data[lo:hi]:
        for c in reasons:
            v = r[h.index(c)]
            if v.isdigit():
                tot[c] = tot.get(c, 0) + int(v)
    s = sum(tot.values())
    print(name, s, ' '.join('%s=%.1f%%' % (k[6:], 100.0 * v / max(s, 1)) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
