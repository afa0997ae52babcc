"""Top SASS lines by stall samples from an ncu source-page CSV (--print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
h = rows[1]
data = rows[2:]
reason = sys.argv[2] if len(sys.argv) > 2 else None
k = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
def tot(r):
    if reason:
        v = r[h.index("stall_" + reason)]
        return int(v) if v.isdigit() else 0
    return sum(int(r[h.index(c)]) for c in cols if r[h.index(c)].isdigit())
idx = sorted(range(len(data)), key=lambda i: -tot(data[i]))[:k]
for i in idx:
    r = data[i]
    top = sorted(((int(r[h.index(c)]) if r[h.index(c)].isdigit() else 0, c[6:]) for c in cols), reverse=True)[:3]
    print("%6d %5d %-60s %s" % (tot(r), i, r[1].strip()[:60], top))
