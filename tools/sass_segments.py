"""Per-region share of stall samples / executed instructions of one kernel in an ncu report
(segments of N SASS instructions, with the source line of the segment's first instruction)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
seg_n = int(sys.argv[3]) if len(sys.argv) > 3 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'Address':
        if hdr is None: hdr = r
        else: break
        continue
    if hdr and r and r[0].startswith('0x'): data.append(r)
iss = hdr.index('Warp Stall Sampling (All Samples)'); iex = hdr.index('Instructions Executed'); isrc = hdr.index('Source')
ts = sum(float(r[iss] or 0) for r in data) or 1; te = sum(float(r[iex] or 0) for r in data) or 1
print(f"{len(data)} SASS, {ts:.0f} samples, {te:.0f} warp-instructions executed")
for a in range(0, len(data), seg_n):
    seg = data[a:a + seg_n]
    s = sum(float(r[iss] or 0) for r in seg); e = sum(float(r[iex] or 0) for r in seg)
    if s / ts > 0.01 or e / te > 0.01:
        top = max(seg, key=lambda r: float(r[iss] or 0))
        print(f"{a:5d} {100*s/ts:5.1f}% samp {100*e/te:5.1f}% inst | {seg[0][isrc][:50]:50s} | hot: {top[isrc][:50]}")
