"""Hot SASS lines of one kernel in an .ncu-rep (dev tool): instruction share and stall share."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if 'Instructions Executed' in r][0]
h = rows[hi]
ie, src, st = h.index('Instructions Executed'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows[hi + 1:]:
    if len(r) <= ie:
        continue
    if r[ie] == 'Instructions Executed':  # next launch's section
        break
    data.append((int(r[ie] or 0), int(r[st] or 0), r[src].strip()))
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
print('total warp instructions', tot, 'stall samples', tots)
for i, (n, s, t) in enumerate(data):
    if n > tot * thr or s > tots * 2 * thr:
        print(f'{i:4d} {n / tot * 100:5.2f}% stall {s / tots * 100:5.2f}%  {t}')
