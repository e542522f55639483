"""SASS executed-instruction attribution by CUDA source line: nvdisasm --print-line-info of the
cubin x the ncu source page (--print-source sass).  usage: sass_attr.py part.dis sass.csv FUNC [OPCODE_PREFIX] [N]"""
import csv, re, collections, sys
dis, sasscsv, fn = sys.argv[1], sys.argv[2], sys.argv[3]
want = sys.argv[4] if len(sys.argv) > 4 else None
lines = open(dis).read().split('\n')
start = None
for i, l in enumerate(lines):
    if l.startswith(fn + ':'): start = i; break
cur = None; addr2 = {}
for l in lines[start+1:]:
    if l.startswith('\t.section') : break
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m: addr2[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(sasscsv)))[2:]
base = int(rows[0][0], 16)
agg = collections.Counter(); aggop = collections.defaultdict(collections.Counter); tot = 0
for r in rows:
    a = int(r[0], 16) - base; ex = float(r[5]); tot += ex
    loc, ins = addr2.get(a, (None, '?'))
    op = ins.split()[0] if not ins.startswith('@') else ins.split()[1]
    if want and not op.startswith(want): continue
    agg[loc] += ex; aggop[loc][op.split('.')[0]] += ex
P = float(__import__("os").environ.get("PAIRS", "2.147455258e9"))
for loc, v in agg.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 30):
    top = ', '.join(f"{o} {c/P:.3f}" for o, c in aggop[loc].most_common(4))
    print(f"{v/P:6.3f} {loc}  [{top}]")
print("total", tot / P)
