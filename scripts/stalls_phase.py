"""Per-phase stall breakdown of an ncu source page (--page source --csv --print-source sass).

Phases are delimited by marker instructions in program order (producer/consumer split at
USETMAXREG.DEALLOC; inside each role a new phase starts at every BAR / SYNCS / LDTM marker).
Prints, per phase, total stall samples, the top reasons, and instruction mix."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
col = {c: i for i, c in enumerate(h)}
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
phases = []
cur = None
for r in data:
    src = r[1].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', src).split(' ')[0]
    marker = any(k in op for k in ('BAR', 'SYNCS', 'USETMAXREG', 'LDTM', 'CALL'))
    if cur is None or marker:
        cur = {'start': r[0][-5:], 'first': src[:40], 'samples': {}, 'ops': {}, 'n': 0}
        phases.append(cur)
    for c in reasons:
        v = r[col[c]]
        if v.isdigit() and int(v):
            cur['samples'][c[6:]] = cur['samples'].get(c[6:], 0) + int(v)
    ex = r[col['Instructions Executed']]
    if ex.isdigit():
        base = op.split('.')[0]
        cur['ops'][base] = cur['ops'].get(base, 0) + int(ex)
        cur['n'] += int(ex)
total = sum(sum(p['samples'].values()) for p in phases)
for p in phases:
    s = sum(p['samples'].values())
    if s < 0.005 * total:
        continue
    top = ' '.join('%s=%.0f%%' % (k, 100.0 * v / s) for k, v in sorted(p['samples'].items(), key=lambda x: -x[1])[:5])
    ops = ' '.join('%s:%d' % (k, v) for k, v in sorted(p['ops'].items(), key=lambda x: -x[1])[:5])
    print('%5s %-40s %5.1f%% | %s | %s' % (p['start'], p['first'], 100.0 * s / total, top, ops))
