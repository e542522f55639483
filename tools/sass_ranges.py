"""Share of stall samples / instructions by source-line range of msp_part.cu (ncu source view)."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
ranges = [tuple(map(int, r.split('-'))) for r in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); fname = ""; hdr = None
tot = [0.0, 0.0]; acc = collections.defaultdict(lambda: [0.0, 0.0]); stalls = collections.defaultdict(lambda: collections.Counter())
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0].isdigit():
        try: smp = float(r[4] or 0); ins = float(r[7] or 0)
        except ValueError: continue
        tot[0] += smp; tot[1] += ins
        key = "other"
        if fname == "msp_part.cu":
            for a, b in ranges:
                if a <= int(r[0]) <= b: key = f"{a}-{b}"
        acc[key][0] += smp; acc[key][1] += ins
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try: stalls[key][h[6:]] += float(r[i] or 0)
                except ValueError: pass
for k, v in sorted(acc.items()):
    top = ", ".join(f"{n} {100*c/max(1,sum(stalls[k].values())):.0f}%" for n, c in stalls[k].most_common(4))
    print(f"{k:10s} {100*v[0]/tot[0]:5.1f}% samples {100*v[1]/tot[1]:5.1f}% instr | {top}")
