"""Summarise an ncu report: duration, issue %, occupancy, top stall reasons, hottest SASS lines."""
import csv, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines()); hdr = next(r); next(r)
    for row in r:
        d = dict(zip(hdr, row))
        def f(v):
            try: return float(v.replace(',', ''))
            except Exception: return None
        items = [(f(v), h) for h, v in d.items() if 'smsp__pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued') and f(v) is not None]
        tot = sum(v for v, h in items) or 1
        top = sorted(items, reverse=True)[:7]
        print(d['Kernel Name'][:24], 'dur_us', d.get('gpu__time_duration.sum'), 'issue%', d.get('sm__inst_issued.avg.pct_of_peak_sustained_active'),
              'occ%', d.get('sm__warps_active.avg.pct_of_peak_sustained_active'),
              'dram_B', float(d.get('dram__bytes_read.sum', '0').replace(',', '') or 0) + float(d.get('dram__bytes_write.sum', '0').replace(',', '') or 0),
              [(h.replace('smsp__pcsamp_warps_issue_stalled_', ''), round(100 * v / tot, 1)) for v, h in top])

def sass(rep, kernel, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    blocks = []; cur = None
    for r in rows:
        if r and r[0] == 'Address':
            cur = {'hdr': r, 'data': []}; blocks.append(cur)
        elif cur is not None and r and r[0].startswith('0x'):
            cur['data'].append(r)
    if not blocks: return
    hdr, data = blocks[0]['hdr'], blocks[0]['data']
    iss = hdr.index('Warp Stall Sampling (All Samples)'); isrc = hdr.index('Source'); iex = hdr.index('Instructions Executed')
    tot = sum(float(r[iss] or 0) for r in data) or 1
    print(kernel, "samples", tot, "instrs", len(data))
    for i, r in sorted(enumerate(data), key=lambda t: -float(t[1][iss] or 0))[:n]:
        print(f"{i:5d} {100*float(r[iss])/tot:5.1f}% ex={r[iex]:>9} {r[isrc][:90]}")

if __name__ == "__main__":
    raw(sys.argv[1])
    for k in sys.argv[2:]:
        sass(sys.argv[1], k)
