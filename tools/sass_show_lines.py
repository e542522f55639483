"""SASS lines of a source-line range with executed counts (per candidate pair).  usage: dis csv FUNC lo hi"""
import csv, re, sys
dis, sasscsv, fn, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
lines = open(dis).read().split('\n')
st = [i for i, l in enumerate(lines) if l.startswith(fn + ':')][0]
cur = None; addr2 = {}
for l in lines[st+1:]:
    if l.startswith('\t.section'): break
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m: addr2[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(sasscsv)))[2:]
base = int(rows[0][0], 16)
P = 2.147455258e9
for r in rows:
    a = int(r[0], 16) - base; ex = float(r[5])
    loc, ins = addr2.get(a, (None, '?'))
    if loc and loc[0] == 'msp_part.cu' and lo <= loc[1] <= hi and ex > P * 0.002:
        print(f"{a:6x} {ex/P:6.3f} {float(r[6])/max(ex,1):5.1f} L{loc[1]} {ins[:80]}")
