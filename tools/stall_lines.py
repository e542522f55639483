"""Top CUDA source lines for one stall reason (ncu source view, summed over SASS of the line)."""
import csv, subprocess, sys, collections
rep, kern, reason = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.defaultdict(lambda: [0.0, ""]); fname = ""; hdr = None; tot = 0.0
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No": hdr = r; idx = hdr.index(reason); continue
    if hdr and r and r[0].isdigit():
        try: v = float(r[idx] or 0)
        except ValueError: continue
        agg[f"{fname}:{r[0]}"][0] += v; agg[f"{fname}:{r[0]}"][1] = r[1][:80]; tot += v
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100*v[0]/max(tot,1):5.1f}%  {k:22s} {v[1]}")
