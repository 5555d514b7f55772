"""Summaries of an ncu report: key metrics per kernel and top stall lines."""
import csv, io, subprocess, sys

rep = sys.argv[1]
want = {'Duration', 'DRAM Throughput', 'Memory Throughput', 'Achieved Occupancy', 'Registers Per Thread',
        'Compute (SM) Throughput', 'L2 Hit Rate', 'Theoretical Occupancy', 'Block Size', 'Grid Size',
        'Executed Ipc Active', 'Dynamic Shared Memory Per Block'}
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
cur = None
for x in r[1:]:
    if x[mi] in want:
        if x[ii] != cur:
            cur = x[ii]
            print('----', x[ii], x[ki][:70])
        print('   ', x[mi], x[vi], x[ui])
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
cols = [i for i, n in enumerate(h) if n in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum', 'Kernel Name')]
units = rr[1]
for x in rr[2:]:
    print(' | '.join(f"{h[i]}={x[i]} {units[i]}" for i in cols)[:300])
if len(sys.argv) > 2:
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                          '-k', sys.argv[2]], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    blocks, curb = [], None
    for row in rows:
        if row and row[0] == 'Kernel Name':
            curb = []
            blocks.append((row[1], curb))
            continue
        if curb is not None:
            curb.append(row)
    for name, b in blocks[:int(sys.argv[3]) if len(sys.argv) > 3 else 1]:
        hh = b[0]
        ai, si, wi, ei = (hh.index(k) for k in ('Address', 'Source', 'Warp Stall Sampling (All Samples)', 'Instructions Executed'))
        data = [(int(x[wi] or 0), x[ai], x[si], x[ei]) for x in b[1:] if len(x) > wi]
        tot = sum(d[0] for d in data)
        print('==', name[:80], 'samples', tot)
        for d in sorted(data, reverse=True)[:30]:
            print(f"{d[0]:6d} {d[3]:>8} {d[2][:110]}")
