"""Per-CUDA-source-line share of stall samples and executed warp instructions (ncu source view)."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0].isdigit():
        d = r
        try:
            samp = float(d[4] or 0); inst = float(d[7] or 0)
        except ValueError:
            continue
        key = f"{fname}:{d[0]}"
        agg[key][0] += samp; agg[key][1] += inst; agg[key][2] = d[1][:70]
ts = sum(v[0] for v in agg.values()) or 1; te = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100*v[0]/ts:5.1f}% samp {100*v[1]/te:5.1f}% inst  {k:22s} {v[2]}")
