"""Build profiles/<tag>_kernels.json (the bench's roofline.traffic source) from one round's captures:
<tag>_prof (k_waves of the second (7,60) s1 solve), <tag>_l1 / <tag>_l2 (level-1 k_scatter and
level-2 k_waves of one huge (9,80) batch).

    python tools/make_kernels_json.py <raw tag in gpurun_out/> <profiles tag> "<code description>"
"""
import csv
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from profile_summary import full  # noqa: E402


def raw_metrics(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    hdr = next(r)
    units = dict(zip(hdr, next(r)))
    row = dict(zip(hdr, next(r)))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "": 1.0, "inst": 1.0}
    val = {}
    for n in names:
        v = float(row[n].replace(",", ""))
        val[n] = v * scale.get(units.get(n, ""), 1.0)
    return val


def main():
    raw, tag, code = sys.argv[1:4]
    g = lambda s: os.path.join("gpurun_out", f"{raw}_{s}.ncu-rep")  # noqa: E731
    _, kw = full(g("prof"), ["k_waves"])
    m = raw_metrics(g("prof"), ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"])
    out = {"k_waves": kw, "traffic": {
        "launch_dram_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
        "dram_read_bytes": m["dram__bytes_read.sum"], "dram_write_bytes": m["dram__bytes_write.sum"],
        "algorithmic_bytes_per_launch": 17179642064,
        "inst_executed": m["smsp__inst_executed.sum"],
        "source": f"ncu --set full --clock-control none of the k_waves launch of tools/rep_solve.py 7 2 (second (7,60) s1 "
                  f"solve = one launch; gpurun_out/{raw}_prof.ncu-rep, {code})"}}
    hb = {"batch": "(9,80) s1 alpha 1117: n_left 2111953682 + n_right 2104980958 keys (tools/run_alpha.py --m 9 --quantile 0.9)"}
    for key, s, k in (("level1_k_scatter_first_launch", "l1", "k_scatter"), ("level2_k_waves", "l2", "k_waves")):
        _, rows = full(g(s), [k])
        x = rows[0]
        mm = raw_metrics(g(s), ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"])
        x.update(dram_read=mm["dram__bytes_read.sum"], dram_write=mm["dram__bytes_write.sum"],
                 inst_executed=mm["smsp__inst_executed.sum"])
        hb[key] = x
    out["huge_batch_9_80_q90"] = hb
    json.dump(out, open(os.path.join("profiles", f"{tag}_kernels.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
