"""Stall-reason totals and top SASS lines of one kernel in an ncu report (instrumentation).
python tools/ncu_stalls.py REPORT KERNEL_REGEX [N]"""
import csv, collections, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                      '-k', 'regex:' + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = [k for k, r in enumerate(rows) if r and r[0] == 'Kernel Name'][0]
h = rows[i + 1]
data = []
for r in rows[i + 2:]:
    if r and r[0] == 'Kernel Name':
        break
    if len(r) == len(h) and r[0].startswith('0x'):
        data.append(r)
st = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
iv = lambda x: int(x) if x.strip().lstrip('-').isdigit() else 0
tot = collections.Counter()
for r in data:
    for c in st:
        tot[c] += iv(r[h.index(c)])
print('stalls:', tot.most_common(8))
si = h.index('Warp Stall Sampling (All Samples)')
ei = h.index('Instructions Executed')
for r in sorted(data, key=lambda r: -iv(r[si]))[:ntop]:
    d = {c: iv(r[h.index(c)]) for c in st}
    top = sorted(d.items(), key=lambda kv: -kv[1])[:2]
    print(f"{iv(r[si]):6d} {r[ei]:>8} {r[0][-5:]} {r[1][:60]:60s} {top}")
