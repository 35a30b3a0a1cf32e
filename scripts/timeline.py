"""Print a compressed per-stream timeline of a chrome trace written by
scripts/gpu_busy.py (TRACE=path): start offset, duration, stream, gap, name."""
import json, sys
d = json.load(open(sys.argv[1]))
ev = [e for e in d['traceEvents'] if e.get('cat') in ('kernel', 'gpu_memcpy', 'gpu_memset') and e.get('ph') == 'X']
ev.sort(key=lambda e: e['ts'])
t0 = ev[0]['ts']
min_dur = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0


def short(n):
    n = n.replace('void ', '').replace('igb::(anonymous namespace)::', '').replace('igb::', '')
    if 'cub::' in n:
        for k in ['Onesweep', 'Histogram', 'ExclusiveSum', 'Select', 'Scan', 'CompactInit', 'ScanInit']:
            if k in n:
                return 'cub:' + k
    return n.split('(')[0][:34]


prev_end = 0.0
for e in ev:
    s = e['ts'] - t0
    du = e['dur']
    gap = s - prev_end
    if du >= min_dur or gap > 15:
        print(f"{s:8.1f} {du:7.1f} s{e['tid']:<3} {'GAP %.0f' % gap if gap > 15 else '':9s} {e.get('cat')[:6]} {short(e['name'])}")
    prev_end = max(prev_end, s + du)
